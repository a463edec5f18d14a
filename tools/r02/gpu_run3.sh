timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --tables gpurun_out/r3_tables.json > gpurun_out/r3_bench_tables.log 2>&1
