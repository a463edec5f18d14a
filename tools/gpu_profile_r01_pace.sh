#!/bin/bash
# after the pacing change: cfg3 / cfg2b fast kernels --set full (one cold launch each), the
# full bench line (with the all-config table) and the bench launch list
mkdir -p gpurun_out
for c in "cfg3 0 f32" "cfg3 1 f32" "cfg2b 0 f32"; do set -- $c
  P="python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 3"
  $P > gpurun_out/plain_$1_k$2_$3.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_$1_k$2_$3 $P > gpurun_out/ncu_$1_k$2_$3.log 2>&1
done
python bench.py > gpurun_out/bench_pace.jsonl 2> gpurun_out/bench_pace.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-table > gpurun_out/ncu_launches.log 2>&1
