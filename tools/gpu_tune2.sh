#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/tune2.log
for rep in 1 2 3; do
 for spec in "4 4 4" "4 2 8" "2 2 8" "2 4 4" "8 2 4"; do
  set -- $spec
  GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 timeout 200 python bench.py --steps 100 --warmup 10 --no-table --e2e-steps 1 --cpu-budget 0.2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('rep$rep R=$1 S=$2 W=$3', 'step %.4f'%d['ms_per_step'], 'fwd %.4f inv %.4f'%(d['kernels']['fast_fwd_ms'], d['kernels']['fast_inv_ms']), 'frac %.4f'%d['roofline']['frac'], 'copy %.0f'%d['roofline']['same_size_copy_gbs'])" >> gpurun_out/tune2.log
 done
done
