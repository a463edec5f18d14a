# r78: tune tests after the test fix; full GPU suite again
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r78_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r78_pytest.log
