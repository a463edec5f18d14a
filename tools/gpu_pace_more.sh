#!/bin/bash
# pacing sweep on the other few-warp FMA configs (tuned geometry, GFT_PACE_NS overrides)
for rep in 1 2; do
for c in "cfg1 0 f32 16777216" "cfg1 1 f32 16777216" "cfg4 0 f64 0" "cfg4 1 f64 0" "cfg2b 0 f32 0"; do set -- $c
  B=""; [ "$4" != "0" ] && B="--batch $4"
  for P in 0 150 300 450 600; do
    GFT_PACE_NS=$P python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 2 $B | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PACE=$P', '$1 k$2 $3', round(d['b2b_gbs']))"
  done
done
done
