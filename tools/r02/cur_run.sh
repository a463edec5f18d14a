# r26: double-buffered A (GFT_TC_A2) in the fp16x2 warp-specialised kernels: parity, burst and sustained A/B
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_right_haar.py tests/test_gpu_filter.py -q -x > gpurun_out/r26_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r26_pytest.log
for p in cfg5b rh0 tr5; do timeout 600 python tools/r02/env_confirm.py $p default GFT_TC_A2=0 >> gpurun_out/r26_burst.log 2>&1; done
timeout 600 python tools/r02/sustain_cmp.py cfg5b 2 default GFT_TC_A2=0 > gpurun_out/r26_sustain.log 2>&1
