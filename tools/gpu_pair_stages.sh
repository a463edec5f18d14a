#!/bin/bash
# pair tcgen05 kernel: tile-buffer count (GFT_TC_PAIR_MAXSTAGES) on n = 80..128 plans
for S in 3 4 5 3 4 5; do
  GFT_TC_PAIR_MAXSTAGES=$S python tools/tc_vs_fma.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['n'] >= 80: print('S<=$S', d['graph'], d['tc']['kernel'][:22], d['tc']['gbs'])
"
done
