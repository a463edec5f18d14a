timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r5_bench.log 2> gpurun_out/r5_bench.err
timeout 900 python -m pytest tests/test_gpu_bench.py tests/test_c_example.py -q > gpurun_out/r5_pytest.log 2>&1
