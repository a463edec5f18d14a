#!/bin/bash
# (experiment, reverted: needed a GFT_TC_MAX_LEAVES knob) n = 64 plans with two 32-node leaves: both on tcgen05 vs only the
# first on tcgen05 and the other as FFMA code in the stager (GFT_TC_MAX_LEAVES=1)
for rep in 1 2; do
for c in "rh0 0" "rh0 1" "ap7 0" "ap9 0" "ap16 0" "ap17 0"; do set -- $c
  for V in 0 1; do
    if [ $V = 1 ]; then export GFT_TC_MAX_LEAVES=1; else unset GFT_TC_MAX_LEAVES; fi
    timeout 300 python tools/profile_kernel.py --config $1 --kind $2 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MAXLEAVES=$V', '$1 k$2', d['kernel'][:30], round(d['b2b_gbs']))"
  done
done
done
