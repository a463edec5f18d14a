#!/bin/bash
# sweep tile size / stages / warps of the FMA skeleton (JIT via NVRTC; kernel names change)
mkdir -p gpurun_out; rm -f gpurun_out/tune.log
for cfg in cfg2; do
 for R in 1 2 4; do for S in 2 3 4 6; do for W in 2 4 8; do
  GFT_TUNE_R=$R GFT_TUNE_STAGES=$S GFT_TUNE_WARPS=$W timeout 120 python tools/profile_kernel.py --config $cfg --kind 0 --iters 12 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ms=sorted(d['ms'][2:]); print('$cfg R=$R S=$S W=$W', d['launch'], 'med %.4f'%ms[len(ms)//2], '%.0f GB/s'%(d['gbs_best']))" >> gpurun_out/tune.log
 done; done; done
done
