# r82: cfg1 @ 2^24 on this box: table (8/3/3/150/2) vs 8 warps, fwd-only and pair streams, both regimes
mkdir -p gpurun_out
L=gpurun_out/r82_cfg1.log; nvidia-smi --query-gpu=uuid --format=csv,noheader > $L
for M in fwd pair; do
SWEEP_MODE=$M SWEEP_BATCH=16777216 python tools/r02/regime_sweep.py cfg1 f32 copy default 8,2,8,150,0 8,3,4,0,0 8,2,8,0,0 >> $L 2>&1
done
