#!/bin/bash
# confirm the cfg3 sweep's best geometries (3 interleaved repetitions, fast fwd/inv, dense fwd)
for rep in 1 2 3; do
  for g in "2 2 10" "3 2 4" "2 3 4" "3 3 4" "2 2 12"; do set -- $g
    for k in 0 1 2; do
      GFT_TUNING_FILE=none GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 python tools/profile_kernel.py --config cfg3 --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R S W = $1 $2 $3 kind $k', round(d['b2b_gbs']))"
    done
  done
done
