# r76: right-Haar 12|20 f64 plan: f64 recipe (16 KiB tiles -> R = 2) vs the table's one-warp CTA
mkdir -p gpurun_out
python tools/r02/rh_f64_sweep.py copy default 2,3,3,600,1 2,3,3,750,1 2,3,3,900,1 2,3,3,450,1 1,3,3,400,1 1,3,3,600,1 2,2,4,0,0 1,2,4,0,0 > gpurun_out/r76_rh_f64.log 2>&1
