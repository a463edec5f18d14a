#!/bin/bash
# Round-1 final evidence (run under gpurun from the repo root): the launch list of the bench
# command (ncu --metrics gpu__time_duration.sum) and one --set full capture of the dominant
# kernel (cfg2 forward), each after the same command exited 0 without ncu.
mkdir -p gpurun_out; rm -f gpurun_out/prof_cfg2_k0_f32.ncu-rep
B="python bench.py --steps 5 --warmup 3 --no-table --e2e-steps 1 --cpu-budget 0.5"
$B > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
P="python tools/profile_kernel.py --config cfg2 --kind 0 --dtype f32 --iters 3"
$P > gpurun_out/plain_cfg2_k0_f32.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_cfg2_k0_f32 $P > gpurun_out/ncu_cfg2_k0_f32.log 2>&1
ls gpurun_out
