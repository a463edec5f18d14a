timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r4_bench.log 2> gpurun_out/r4_bench.err
timeout 900 python bench.py --steps 20 --warmup 5 --tables gpurun_out/r4_tables.json > gpurun_out/r4_bench_tables.log 2>&1
