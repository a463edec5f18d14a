# r38: extended randomised parity sweep (seeds 40..299) over the session-3 kernels
GFT_FUZZ_SEEDS=40:300 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q -k random_plan_parity > gpurun_out/r38_fuzz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r38_fuzz.log
