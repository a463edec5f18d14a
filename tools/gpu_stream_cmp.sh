#!/bin/bash
# streamed leaf outputs (GFT_STREAM=1) vs register-resident y (GFT_STREAM=0), back to back
for V in 1 0 1 0; do
  for c in "cfg4 0 f64" "cfg4 1 f64" "cfg4 2 f64" "cfg5b 2 f32" "cfg4 0 f32"; do set -- $c
    GFT_STREAM=$V python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('STREAM=$V', '$1 k$2 $3', d['kernel'][:24], round(d['b2b_gbs']))"
  done
done
