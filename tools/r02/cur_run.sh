# r37: max-size (n = 256) parity test
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "max_size" > gpurun_out/r37_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r37_pytest.log
