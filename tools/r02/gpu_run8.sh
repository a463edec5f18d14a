# session-2 re-entry validation: GPU suite, smoke, the driver's bench command
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r8_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r8_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r8_tables.json > gpurun_out/r8_bench.log 2> gpurun_out/r8_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r8_ref.log 2>&1
