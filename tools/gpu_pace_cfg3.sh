#!/bin/bash
# cfg3 pacing sweep: __nanosleep(GFT_PACE_NS) per warp tile before the store, fwd and inv
for rep in 1 2; do
for g in "3 3 4" "2 3 4" "3 2 4" "4 2 4" "2 3 5" "3 3 5" "2 4 4"; do set -- $g
  for P in 0 200 250 300 350 400 500; do
    for k in 0 1; do
      GFT_PACE_NS=$P GFT_TUNING_FILE=none GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 python tools/profile_kernel.py --config cfg3 --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PACE=$P geo $1 $2 $3 kind $k', round(d['b2b_gbs']))"
    done
  done
done
done
