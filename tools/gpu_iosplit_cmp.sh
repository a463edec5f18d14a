#!/bin/bash
# cfg5b / n=96..128 plans: IO-split warp-specialised kernel (default) vs plain pair kernel
for V in 0 1 0 1; do
  if [ $V = 0 ]; then export GFT_TC_IOSPLIT=1; else unset GFT_TC_IOSPLIT; fi
  for c in "cfg5b 0" "cfg5b 1"; do set -- $c
    python tools/profile_kernel.py --config $1 --kind $2 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_SPLIT=$V', '$1 k$2', d['kernel'][:24], round(d['b2b_gbs']))"
  done
  python tools/tc_vs_fma.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['n'] >= 80: print('NO_SPLIT=$V', d['graph'], d['tc']['kernel'][:24], d['tc']['gbs'])
"
done
