mkdir -p gpurun_out
GFT_PDL=0 timeout 300 python bench.py --steps 100 --warmup 10 --no-table --e2e-steps 1 --cpu-budget 0.5 > gpurun_out/bench_nopdl.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-table --e2e-steps 1 --cpu-budget 0.5 > gpurun_out/bench_pdl.log 2>&1
for cfg in cfg4 cfg5b; do
GFT_PDL=0 timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --no-table --e2e-steps 1 --cpu-budget 0.5 > gpurun_out/bench_nopdl_$cfg.log 2>&1
timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --no-table --e2e-steps 1 --cpu-budget 0.5 > gpurun_out/bench_pdl_$cfg.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
