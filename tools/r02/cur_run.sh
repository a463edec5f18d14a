# r70: side tables with the SURVEY 8(d) estimator (5 warm-up + 5 x 10 calls, median and min)
mkdir -p gpurun_out
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r70_tables.json > gpurun_out/r70_bench_tables.log 2> gpurun_out/r70_bench_tables.err; echo "rc=$?" >> gpurun_out/r70_bench_tables.err
timeout 600 python -m pytest tests/test_gpu_bench.py -q > gpurun_out/r70_pytest_bench.log 2>&1
