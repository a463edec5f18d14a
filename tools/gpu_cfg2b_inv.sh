#!/bin/bash
# cfg2b inverse geometry probe (the forward's tuned 4/2/8 vs alternatives)
for G in "4 2 8" "2 2 8" "4 3 4" "8 2 4" "2 3 8" "4 2 4"; do set -- $G
  for k in 0 1; do
    GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 GFT_TUNING_FILE=none python tools/profile_kernel.py --config cfg2b --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $3 k$k', round(d['b2b_gbs']))"
  done
done
