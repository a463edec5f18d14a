# re-entry validation (fresh container): full GPU suite, smoke, driver bench command
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r10_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r10_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r10_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r10_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r10_tables.json > gpurun_out/r10_bench.log 2> gpurun_out/r10_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r10_ref.log 2>&1
