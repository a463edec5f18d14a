# r56: tune tests (incl. GFT_TUNE_SUSTAINED), abi tests, bench at the new cfg5a inverse geometry
mkdir -p gpurun_out
L=gpurun_out/r56.log; : > $L
timeout 900 python -m pytest tests/test_gpu_tune.py tests/test_gpu_parity.py -q -x >> $L 2>&1; echo "pytest rc=$?" >> $L
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r56_bench.log 2> gpurun_out/r56_bench.err; echo "bench rc=$?" >> $L
