#!/bin/bash
# Re-profile the FMA-skeleton kernels whose hashes changed with the pacing change (cfg2,
# cfg4 f32/f64, cfg5a, cfg5b dense, cfg1 at 2^24), the right-Haar / approximate rows and the
# bench launch list.  Each ncu capture runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
for spec in "cfg2 0 f32" "cfg2 1 f32" "cfg4 0 f32" "cfg4 0 f64" "cfg5a 0 f32" "cfg5b 2 f32"; do
  set -- $spec
  P="python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 3"
  $P > gpurun_out/plain_$1_k$2_$3.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_$1_k$2_$3 $P > gpurun_out/ncu_$1_k$2_$3.log 2>&1
done
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
