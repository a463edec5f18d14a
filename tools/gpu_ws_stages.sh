#!/bin/bash
# warp-specialised tcgen05 kernel: tile-buffer count sweep (GFT_TC_WS_STAGES)
for S in 4 5 6 4 5 6; do
  GFT_TC_WS_STAGES=$S python tools/tc_vs_fma.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['n'] < 128: print('S=$S', d['graph'], d['tc']['kernel'][:20], d['tc']['gbs'])
"
done
