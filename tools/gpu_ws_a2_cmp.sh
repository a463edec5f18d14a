#!/bin/bash
# warp-specialised tcgen05 kernel: A operand double-buffered in TMEM (opt-in GFT_TC_WS_A2=1)
# vs one A buffer (default); n = 64 plans; then the tensor-core parity tests
mkdir -p gpurun_out
{
for spec in rh0 ap7 ap9 ap16; do
  for k in 0 1; do
    for v in "A2" "A1"; do
      if [ $v = A2 ]; then export GFT_TC_WS_A2=1; else unset GFT_TC_WS_A2; fi
      timeout 120 python tools/profile_kernel.py --config $spec --kind $k --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec k$k $v', d['kernel'], round(d['b2b_ms']*1000,2), 'us', round(d['b2b_gbs']))"
    done
  done
done
unset GFT_TC_WS_A2
} > gpurun_out/ws_a2_cmp.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_right_haar.py tests/test_gpu_approx.py -q -k "tensor or tc or right or approx" > gpurun_out/ws_a2_tests.log 2>&1; echo rc=$? >> gpurun_out/ws_a2_tests.log
