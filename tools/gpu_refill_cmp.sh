#!/bin/bash
# early refill experiment (measured -5..-9%, removed; see profiles/r01/autotune/refill_cmp.log).
# Needs the GFT_REFILL_EARLY skeleton variant, which is no longer in the tree.
# vs the default (the previous iteration's buffer is reloaded), FMA skeleton, back to back;
# with the tuned geometry and with one more stage
for rep in 1 2; do
for c in "cfg2 0 f32" "cfg3 0 f32" "cfg4 0 f32" "cfg4 0 f64" "cfg5a 0 f32" "cfg2 1 f32" "cfg3 1 f32"; do set -- $c
  for V in 0 1; do
    for ST in "" 3 4; do
      GFT_REFILL_EARLY=$V GFT_TUNE_STAGES=$ST python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('REFILL=$V S=${ST:-tuned}', '$1 k$2 $3', d['kernel'][:26], round(d['b2b_gbs']))"
    done
  done
done
done
