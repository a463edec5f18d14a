#!/bin/bash
# ncu --set full of the tcgen05 3xTF32 fast kernels (cfg5b fwd / inv)
mkdir -p gpurun_out
for spec in "cfg5b 0" "cfg5b 1"; do
  set -- $spec
  P="python tools/profile_kernel.py --config $1 --kind $2 --iters 3"
  $P > gpurun_out/plain_$1_k$2.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_$1_k$2_tc $P > gpurun_out/ncu_$1_k$2.log 2>&1
done
