# r81: final validation after cfg2 moved to the sustained-regime geometry (GPU suite, smoke, driver bench, reference arm, side tables)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r81_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r81_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r81_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r81_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r81_bench.log 2> gpurun_out/r81_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r81_ref.log 2>&1
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r81_tables.json > gpurun_out/r81_bench_tables.log 2>&1
