set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi0.csv
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r1_bench.log 2> gpurun_out/r1_bench.err; echo "bench rc=$?" >> gpurun_out/r1_bench.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --tables gpurun_out/r1_tables.json > gpurun_out/r1_bench_tables.log 2>&1
