#!/bin/bash
# tensor-core kernel variants on the side-table tcgen05 plans, back to back: default
# (warp-specialised for n <= 64), pair with two warpgroups, plain pair, single CTA
for rep in 1 2; do
for c in "rh0 0" "ap7 0" "ap9 0" "ap16 0" "ap17 0" "rh1 0" "cfg5b 0"; do set -- $c
  for V in default nows nows2wg nopair; do
    unset GFT_NO_TC_WS GFT_NO_TC_2WG GFT_NO_CTA_PAIR
    case $V in nows) export GFT_NO_TC_WS=1;; nows2wg) export GFT_NO_TC_WS=1 GFT_NO_TC_2WG=1;; nopair) export GFT_NO_CTA_PAIR=1;; esac
    timeout 300 python tools/profile_kernel.py --config $1 --kind $2 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', '$1 k$2', d['kernel'][:30], round(d['b2b_gbs']))"
  done
done
done
