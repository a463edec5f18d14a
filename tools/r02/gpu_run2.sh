set -x
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2> gpurun_out/r2_bench.err; echo "bench rc=$?" >> gpurun_out/r2_bench.err
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 300 python tools/r02/tc_probe.py rh0 > gpurun_out/r2_probe.log 2>&1
timeout 300 python tools/r02/tc_probe.py cfg5b >> gpurun_out/r2_probe.log 2>&1
