# r59: extended randomised parity sweep, seeds 300..800 (500 new random plans)
mkdir -p gpurun_out
GFT_FUZZ_SEEDS=300:800 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/r59_fuzz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r59_fuzz.log
