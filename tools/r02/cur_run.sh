# r65: per-warp store rate limit, spinning on %globaltimer (32 ns resolution)
mkdir -p gpurun_out
L=gpurun_out/r65_rate_spin.log; nvidia-smi --query-gpu=uuid --format=csv,noheader > $L
python tools/r02/regime_sweep.py cfg4 f32 copy default 1,3,3,0,2,700 1,3,3,0,2,800 1,3,3,0,2,900 1,3,3,0,2,1000 1,3,3,0,2,1100 1,2,8,0,0,2200 1,2,8,0,0,2500 1,2,8,0,0,2700 1,2,8,0,0,2900 1,2,8,0,0,3100 >> $L 2>&1
python tools/r02/regime_sweep.py cfg2 f32 copy default 4,3,3,0,2,800 4,3,3,0,2,900 4,3,3,0,2,1000 4,3,3,0,2,1100 4,2,8,0,0,2500 4,2,8,0,0,2800 4,2,8,0,0,3000 >> $L 2>&1
SWEEP_ROUNDS=2 python tools/r02/step_sweep2.py copy default "fwd=1,2,8,0,0,2400;inv=1,2,8,0,0,2400" "fwd=1,2,8,0,0,2700;inv=1,2,8,0,0,2700" "fwd=1,2,8,0,0,2900;inv=1,2,8,0,0,2900" "fwd=1,2,8,0,0,3100;inv=1,2,8,0,0,3100" >> $L 2>&1
