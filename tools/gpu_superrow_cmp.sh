#!/bin/bash
# odd-pitch configs: super-row TMA tensor mode (GFT_SUPERROW=1) vs 1-D bulk copies (default)
for V in 0 1 0 1; do
  if [ $V = 0 ]; then export GFT_SUPERROW=1; else unset GFT_SUPERROW; fi
  for k in 0 1; do
    python tools/profile_kernel.py --config cfg3 --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_SUPERROW=$V cfg3 k$k', d['kernel'][:22], round(d['b2b_gbs']))"
  done
done
