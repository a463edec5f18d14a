#!/bin/bash
# L2 promotion of the signal tensor maps (GFT_L2PROMO = 0 / 128 / 256), back to back
for rep in 1 2; do
for c in "cfg2 0 f32" "cfg4 0 f32" "cfg4 0 f64" "cfg5a 0 f32" "cfg5b 0 f32" "cfg2b 0 f32"; do set -- $c
  for V in 256 128 0; do
    GFT_L2PROMO=$V python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PROMO=$V', '$1 k$2 $3', round(d['b2b_gbs']))"
  done
done
done
