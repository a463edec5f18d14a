#!/bin/bash
# packed-view TMA mode (GFT_PACK) vs narrow boxes: n = 8 (cfg1 at 2^24) and n = 16 (cfg2)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -k packed_view > gpurun_out/pack_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pack_tests.log
run() {  # label env...
  for k in 0 1; do
    env "$@" GFT_TUNING_FILE=${TF:-} timeout 120 python tools/profile_kernel.py --config $CFG --kind $k --iters 2 --batch $B | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG k$k', '$*', round(d['b2b_ms']*1000,2), 'us', round(d['b2b_gbs']))"
  done
}
{
CFG=cfg1 B=16777216
for G in "2 2 8" "4 2 8" "8 2 8" "4 2 4" "8 2 4" "8 3 4" "4 3 8"; do set -- $G
  run GFT_PACK=1 GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3
done
run GFT_PACK=0
CFG=cfg1 B=4096
run GFT_PACK=1
run GFT_PACK=0
CFG=cfg2 B=4194304
run GFT_PACK=0
run GFT_PACK=1
for G in "2 2 8" "8 2 8" "4 2 4"; do set -- $G
  run GFT_PACK=1 GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3
done
} > gpurun_out/pack_cmp.log 2>&1
