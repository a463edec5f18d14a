#!/bin/bash
# pair tcgen05 kernel: per-chunk `staged` signals (default) vs one per leaf (GFT_TC_STAGED_LEAF=1)
for V in 0 1 0 1; do
  if [ $V = 1 ]; then export GFT_TC_STAGED_LEAF=1; else unset GFT_TC_STAGED_LEAF; fi
  for k in 0 1; do
    python tools/profile_kernel.py --config cfg5b --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ONCE=$V cfg5b k$k', d['kernel'][:24], round(d['b2b_gbs']))"
  done
  python tools/tc_vs_fma.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['n'] >= 80: print('ONCE=$V', d['graph'], d['tc']['kernel'][:24], d['tc']['gbs'])
"
done
