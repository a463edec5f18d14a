#!/bin/bash
# ncu evidence for the kernels the bench reports (run under gpurun from the repo root)
mkdir -p gpurun_out; rm -f gpurun_out/prof_*.ncu-rep
B="python bench.py --steps 5 --warmup 3 --no-table --e2e-steps 1 --cpu-budget 0.5"
$B > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
for spec in "cfg2 0 f32" "cfg2 1 f32" "cfg3 0 f32" "cfg4 0 f32" "cfg4 0 f64" "cfg5a 0 f32" "cfg5b 0 f32" "cfg5b 1 f32" "cfg5b 2 f32"; do
  set -- $spec
  P="python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 3"
  $P > gpurun_out/plain_$1_k$2_$3.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_$1_k$2_$3 $P > gpurun_out/ncu_$1_k$2_$3.log 2>&1
done
ls gpurun_out
