#!/bin/bash
# pacing experiment: __nanosleep(GFT_PACE_NS) per warp tile before the store is issued
for rep in 1 2; do
for c in "cfg3 0 f32 2 2 10" "cfg3 0 f32 3 3 4" "cfg2 0 f32 4 2 8" "cfg5a 0 f32 1 2 8" "cfg4 0 f32 2 2 4"; do set -- $c
  for P in 0 100 300 600 1000; do
    GFT_PACE_NS=$P GFT_TUNING_FILE=none GFT_TUNE_R=$4 GFT_TUNE_STAGES=$5 GFT_TUNE_WARPS=$6 python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PACE=$P', '$1 k$2 $3 geo $4 $5 $6', round(d['b2b_gbs']))"
  done
done
done
