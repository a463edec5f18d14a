#!/bin/bash
# sweep tile rows per thread (R) / stages (S) / warps per CTA (W) of the FMA skeleton
mkdir -p gpurun_out; rm -f gpurun_out/tune.log
run() {  # cfg dtype R S W
  GFT_TUNE_R=$3 GFT_TUNE_STAGES=$4 GFT_TUNE_WARPS=$5 timeout 120 python tools/profile_kernel.py --config $1 --dtype $2 --kind 0 --iters 3 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('$1 $2 R=$3 S=$4 W=$5', d['launch'], 'b2b %.4f'%d['b2b_ms'], '%.0f GB/s'%d['b2b_gbs'])" >> gpurun_out/tune.log
}
for cfg in cfg2 cfg3 cfg5a; do
  run $cfg f32 0 0 0
  for R in 2 4 8; do for W in 4 8 16; do for S in 2 3; do run $cfg f32 $R $S $W; done; done; done
done
run cfg4 f32 0 0 0; run cfg4 f32 2 2 8; run cfg4 f32 2 3 8; run cfg4 f32 4 2 8; run cfg4 f32 1 4 8; run cfg4 f32 2 2 16
run cfg4 f64 0 0 0; run cfg4 f64 1 2 8; run cfg4 f64 2 2 8; run cfg4 f64 1 3 8
