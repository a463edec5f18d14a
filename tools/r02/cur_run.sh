# r71: last validation at the final HEAD (GPU suite, smoke, driver bench, reference arm)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r71_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r71_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r71_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r71_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r71_bench.log 2> gpurun_out/r71_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r71_ref.log 2>&1
