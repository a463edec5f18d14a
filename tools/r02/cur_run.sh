# r43: maximum-size edge cases (buffers > 4 GiB, batch > 2^30 rows) on the B200
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv > gpurun_out/r43_large.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_large.py -q -x --durations=10 >> gpurun_out/r43_large.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r43_large.log
