# r68: forward-only / inverse-only streams (not pairs) for the few-warp paced geometries, both regimes
mkdir -p gpurun_out
L=gpurun_out/r68_fwd_only.log; nvidia-smi --query-gpu=uuid --format=csv,noheader > $L
for M in fwd inv pair; do
SWEEP_MODE=$M SWEEP_BATCH=16777216 python tools/r02/regime_sweep.py cfg1 f32 copy default 8,2,8,150,0 8,3,4,0,0 8,3,3,100,2 8,3,3,200,2 >> $L 2>&1
done
for M in fwd inv; do
SWEEP_MODE=$M python tools/r02/regime_sweep.py cfg2 f32 copy default 4,2,8,0,0 >> $L 2>&1
SWEEP_MODE=$M python tools/r02/regime_sweep.py cfg4 f32 copy default 1,2,8,0,0 >> $L 2>&1
SWEEP_MODE=$M python tools/r02/regime_sweep.py cfg3 f32 copy default 4,2,6,0,0 >> $L 2>&1
done
