#!/bin/bash
# (experiment, reverted) IO-split warp-specialised kernel at n = 64 (input ring + one output buffer, storer
# warp) vs the default warp-specialised kernel on the n = 64 tensor-core plans, back to back
for rep in 1 2; do
for c in "rh0 0" "rh0 1" "ap7 0" "ap9 0" "ap16 0" "ap17 0" "cfg5b 0"; do set -- $c
  for V in "" 1; do
    GFT_TC_IOSPLIT=$V timeout 300 python tools/profile_kernel.py --config $1 --kind $2 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('IOSPLIT=${V:-0}', '$1 k$2', d['kernel'][:30], round(d['b2b_gbs']))"
  done
done
done
