#!/bin/bash
# back-to-back cfg5b forward: WS-split vs pair kernel, with and without programmatic dependent launch
for P in 1 0; do
  for V in 0 1; do
    if [ $V = 0 ]; then export GFT_TC_IOSPLIT=1; else unset GFT_TC_IOSPLIT; fi
    GFT_PDL=$P python tools/profile_kernel.py --config cfg5b --kind 0 --iters 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=$P NO_SPLIT=$V', d['kernel'][:24], 'b2b', round(d['b2b_gbs']), 'single', [round(x,4) for x in d['ms'][1:]])"
  done
done
