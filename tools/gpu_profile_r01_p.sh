#!/bin/bash
# Re-profile after the packed-view / approx-on-tcgen05 changes (kernel hashes changed):
# f64 n=32 geometry sweep (right-Haar case rh3), ncu --set full of every config's kernels,
# the bench launch list, and the right-Haar / approximate kernels.  Each ncu capture runs
# only after the same command exited 0 without ncu.
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
for G in "1 2 8" "1 3 8" "1 2 6" "2 2 4" "1 3 6" "1 4 4" "2 3 3"; do set -- $G
  GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 timeout 120 python tools/profile_kernel.py --config rh3 --kind 0 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rh3 $1 $2 $3', round(d['b2b_ms']*1000,2), 'us', round(d['b2b_gbs']))"
done > gpurun_out/rh3_geo.log 2>&1
bash tools/gpu_profile_r01_all.sh > gpurun_out/profile_all.log 2>&1
P="python tools/profile_kernel.py --config cfg1 --kind 0 --dtype f32 --iters 3 --batch 16777216"
$P > gpurun_out/plain_cfg1big.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_cfg1big_k0_f32 $P > gpurun_out/ncu_cfg1big.log 2>&1
M="python tools/profile_many.py rh0:0 rh1:0 rh3:0 ap7:0 ap8:0 ap16:0"
$M > gpurun_out/plain_many.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gft_ -c 12 -o gpurun_out/prof_next_rows $M > gpurun_out/ncu_many.log 2>&1
B="python bench.py --steps 5 --warmup 3 --no-table --e2e-steps 1 --cpu-budget 0.5"
$B > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out/*.ncu-rep
