#!/bin/bash
# persistence GPU test + n=8 geometry at 2^24 signals
mkdir -p gpurun_out
python -m pytest tests/test_plan_persistence.py -q -m gpu > gpurun_out/persist.log 2>&1; echo "persist rc=$?" >> gpurun_out/persist.log
for G in "2 2 8" "4 2 8" "8 2 8" "8 2 4" "4 3 8" "8 3 4" "16 2 4" "4 2 16" "8 2 16"; do set -- $G
  for B in 4096 16777216; do
    GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 GFT_TUNING_FILE=none timeout 120 python tools/profile_kernel.py --config cfg1 --kind 0 --iters 2 --batch $B | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $3', $B, round(d['b2b_ms']*1000,2), 'us', round(d['b2b_gbs']))"
  done
done > gpurun_out/cfg1_geo.log 2>&1
