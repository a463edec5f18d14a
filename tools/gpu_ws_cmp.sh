#!/bin/bash
# back-to-back GB/s of the tcgen05 plans: warp-specialised (default) vs plain pair kernel
for V in 0 1 0 1; do
  if [ $V = 1 ]; then export GFT_NO_TC_WS=1; else unset GFT_NO_TC_WS; fi
  for c in "cfg5b 0" "cfg5b 1"; do set -- $c
    python tools/profile_kernel.py --config $1 --kind $2 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_WS=$V', '$1 k$2', d['kernel'][:24], round(d['b2b_gbs']), [round(x,4) for x in d['ms']])"
  done
  python tools/tc_vs_fma.py 2>/dev/null | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_WS=$V', d['graph'], d['tc']['kernel'][:24], d['tc']['gbs'])"
done
