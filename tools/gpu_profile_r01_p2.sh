#!/bin/bash
# the dominant kernel (cfg2 forward) --set full capture + more f64 n=32 geometries
mkdir -p gpurun_out
P="python tools/profile_kernel.py --config cfg2 --kind 0 --dtype f32 --iters 3"
$P > gpurun_out/plain_cfg2_k0_f32.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_cfg2_k0_f32 $P > gpurun_out/ncu_cfg2_k0_f32.log 2>&1
for G in "1 4 4" "1 2 6" "1 3 4" "1 2 4" "1 4 3" "1 5 4" "1 6 3" "1 3 5" "1 4 5" "1 2 5"; do set -- $G
  for k in 0 1; do
  GFT_TUNE_R=$1 GFT_TUNE_STAGES=$2 GFT_TUNE_WARPS=$3 timeout 120 python tools/profile_kernel.py --config rh3 --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rh3 k$k $1 $2 $3', round(d['b2b_ms']*1000,2), 'us', round(d['b2b_gbs']))"
  done
done > gpurun_out/rh3_geo2.log 2>&1
