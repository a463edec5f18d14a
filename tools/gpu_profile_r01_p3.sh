#!/bin/bash
# after the WS skeleton change: tests touching it, the C example, smoke, and a fresh ncu
# capture of the right-Haar / approximate kernels (tc3 hashes changed; rh3 new geometry)
mkdir -p gpurun_out; rm -f gpurun_out/prof_next_rows.ncu-rep
python -m pytest tests/test_gpu_parity.py tests/test_c_example.py tests/test_gpu_right_haar.py tests/test_gpu_approx.py -q > gpurun_out/p3_tests.log 2>&1; echo rc=$? >> gpurun_out/p3_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
M="python tools/profile_many.py rh0:0 rh1:0 rh3:0 ap7:0 ap8:0 ap16:0"
$M > gpurun_out/plain_many.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gft_ -c 12 -o gpurun_out/prof_next_rows $M > gpurun_out/ncu_many.log 2>&1
ls -la gpurun_out/prof_next_rows.ncu-rep
