# tab:runtime side table with the tcgen05 dense comparison at n = 80 too
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r16_tables.json > gpurun_out/r16_bench.log 2> gpurun_out/r16_bench.err
