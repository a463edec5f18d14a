#!/bin/bash
# cfg1 geometry at its own batch (4096, launch-bound) and at 2^24 signals (bandwidth)
for G in "2 2 8" "4 2 8" "8 2 8" "8 3 4" "4 3 8"; do set -- $G
  for B in 4096 16777216; do
    GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 GFT_TUNING_FILE=none python tools/profile_kernel.py --config cfg1 --kind 0 --iters 2 --batch $B | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $3', $B, round(d['b2b_ms']*1000,2), 'us', round(d['b2b_gbs']))"
  done
done
