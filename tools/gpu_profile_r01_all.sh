#!/bin/bash
# ncu --set full of every config's fast kernels (+ cfg5b dense) with the current code, one
# process per capture, each after the same command exited 0 without ncu (run under gpurun)
mkdir -p gpurun_out
for spec in "cfg2 1 f32" "cfg2b 0 f32" "cfg3 0 f32" "cfg4 0 f32" "cfg4 0 f64" "cfg5a 0 f32" "cfg5b 0 f32" "cfg5b 1 f32" "cfg5b 2 f32"; do
  set -- $spec
  P="python tools/profile_kernel.py --config $1 --kind $2 --dtype $3 --iters 3"
  $P > gpurun_out/plain_$1_k$2_$3.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_$1_k$2_$3 $P > gpurun_out/ncu_$1_k$2_$3.log 2>&1
done
ls gpurun_out/*.ncu-rep
