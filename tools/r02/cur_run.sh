# r63: rate-limited 8-warp cfg5a kernels inside the headline step (both regimes)
mkdir -p gpurun_out
L=gpurun_out/r63_rate_step.log; nvidia-smi --query-gpu=uuid --format=csv,noheader > $L
SWEEP_ROUNDS=2 python tools/r02/step_sweep2.py copy default "fwd=1,2,8,0,0,900;inv=1,2,8,0,0,900" "fwd=1,2,8,0,0,1900;inv=1,2,8,0,0,1900" "fwd=1,2,8,0,0,2900;inv=1,2,8,0,0,2900" "fwd=1,2,8,0,0,3900;inv=1,2,8,0,0,3900" "fwd=1,2,8,0,0,2900" "inv=1,2,8,0,0,2900" "fwd=1,3,8,0,0,2900;inv=1,3,8,0,0,2900" >> $L 2>&1
python tools/r02/regime_sweep.py cfg4 f32 copy default 1,2,8,0,0,900 1,2,8,0,0,1900 1,2,8,0,0,2900 1,2,8,0,0,3900 1,3,8,0,0,2900 1,2,12,0,0,3900 >> $L 2>&1
