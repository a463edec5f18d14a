timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r7_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r7_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r7_bench.log 2> gpurun_out/r7_bench.err
timeout 600 python tools/r02/tc_probe.py rh0 2 > gpurun_out/r7_probe.log 2>&1
GFT_TC_F16=0 timeout 600 python tools/r02/tc_probe.py rh0 2 >> gpurun_out/r7_probe.log 2>&1
