# r41: bench contract test + driver command with the sustained copy arm
timeout 900 python -m pytest tests/test_gpu_bench.py -q > gpurun_out/r41_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r41_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r41_bench.log 2> gpurun_out/r41_bench.err
