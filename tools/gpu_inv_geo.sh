for G in "2 2 4" "1 2 8" "1 3 4" "2 3 4" "1 2 12"; do set -- $G
  for c in "cfg4 f32" "cfg2b f32" "cfg5a f32"; do set -- $G $c
    GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 GFT_TUNING_FILE=none python tools/profile_kernel.py --config $4 --dtype $5 --kind 1 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $3', '$4 inv', round(d['b2b_gbs']))"
  done
done
