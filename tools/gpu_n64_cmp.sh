#!/bin/bash
# n = 64 tensor-core plans: warp-specialised kernel (default) vs pair kernel with 4 / 6 buffers
run() { python tools/tc_vs_fma.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['n'] == 64: print('$1', d['graph'], d['tc']['kernel'][:22], d['tc']['gbs'])
"; }
for rep in 1 2; do
  run WS
  GFT_NO_TC_WS=1 GFT_NO_TC_2WG=1 GFT_TC_PAIR_MAXSTAGES=4 run pair4
  GFT_NO_TC_WS=1 GFT_NO_TC_2WG=1 GFT_TC_PAIR_MAXSTAGES=6 run pair6
  GFT_NO_TC_WS=1 GFT_TC_PAIR_MAXSTAGES=6 run 2wg6
done
