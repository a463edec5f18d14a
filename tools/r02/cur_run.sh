# r39: randomised parity sweep seeds 0..299 with the split kernel-exactness / basis-conditioning checks
GFT_FUZZ_SEEDS=0:300 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/r39_fuzz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r39_fuzz.log
