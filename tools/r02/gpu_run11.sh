# e2e run-to-run variation; IO-split tcgen05 kernel at n = 64 (rh0); geometry sweeps of cfg1@2^24 fwd
# and the right-Haar 12|20 f64 plan; ncu --set full of the default rh0 forward
out=gpurun_out/r11_e2e.log; : > $out
for c in 131072 262144 65536; do E2E_CHUNK=$c timeout 300 python tools/r02/e2e_var.py >> $out 2>&1; done
timeout 600 python tools/r02/env_confirm.py rh0 default GFT_TC_IOSPLIT=1 GFT_TC_IOSPLIT=1,GFT_TC_IOSPLIT_STAGES=3 \
   GFT_TC_IOSPLIT=1,GFT_TC_IOSPLIT_STAGES=4 > gpurun_out/r11_rh0_io.log 2>&1
SWEEP_R=4,8 SWEEP_WARPS=3,4,8 SWEEP_PACE=0,150 SWEEP_OBUF=0,2 timeout 900 python tools/r02/geo_sweep.py cfg1@24 fwd > gpurun_out/r11_sweep.log 2>&1
SWEEP_R=1,2,4 SWEEP_WARPS=1,2,3,4,8 SWEEP_PACE=0,150 SWEEP_OBUF=0,2 timeout 900 python tools/r02/geo_sweep.py rh3 fwd >> gpurun_out/r11_sweep.log 2>&1
SWEEP_R=1,2,4 SWEEP_WARPS=1,2,3,4,8 SWEEP_PACE=0,150 SWEEP_OBUF=0,2 timeout 900 python tools/r02/geo_sweep.py rh3 inv >> gpurun_out/r11_sweep.log 2>&1
timeout 300 python tools/profile_kernel.py --config rh0 --kind 0 --iters 3 > gpurun_out/r11_rh0_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gft_ -s 2 -c 1 -o gpurun_out/r11_rh0_fwd \
    python tools/profile_kernel.py --config rh0 --kind 0 --iters 3 > gpurun_out/r11_rh0_ncu.log 2>&1
