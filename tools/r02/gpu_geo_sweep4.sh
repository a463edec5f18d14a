out=gpurun_out/r02_geo_sweep4.log
: > $out
SWEEP_R=1,2 SWEEP_WARPS=2,3,4,6,8 SWEEP_OBUF=0,2 SWEEP_PACE=0,50,100,150,250 timeout 2400 python tools/r02/geo_sweep.py cfg5a fwd >> $out 2>&1
