for rep in 1 2; do
for G in "1 2 8" "2 2 4" "1 3 4"; do set -- $G
for C in "cfg4 2097152" "cfg4 1048576" "cfg5a 2097152" "cfg5a 1048576"; do set -- $G $C
GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 GFT_TUNING_FILE=none python tools/profile_kernel.py --config $4 --dtype f32 --kind 0 --iters 2 --batch $5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $3', '$4', $5, round(d['b2b_gbs']))"
done; done; done
