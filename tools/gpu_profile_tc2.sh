#!/bin/bash
mkdir -p gpurun_out
P="python tools/profile_kernel.py --config cfg5b --kind 0 --iters 3"
$P > gpurun_out/plain_tc2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gft_ -s 1 -c 1 -o gpurun_out/prof_cfg5b_k0_tc2 $P > gpurun_out/ncu_tc2.log 2>&1
