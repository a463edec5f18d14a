# bench side tables incl. the tab:runtime re-timing and the oracle CPU table
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r15_tables.json > gpurun_out/r15_bench.log 2> gpurun_out/r15_bench.err
