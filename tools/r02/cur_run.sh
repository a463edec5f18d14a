# r24: bench (driver command + side tables) after split-store and the IO-split dense n = 128 kernel; steady-state ncu traffic of the new kernel names
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r24_bench.log 2> gpurun_out/r24_bench.err
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r24_tables.json > gpurun_out/r24_bench_t.log 2> gpurun_out/r24_bench_t.err
python tools/r02/profile_steady.py cfg5a cfg5b rh0 > gpurun_out/r24_steady_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --cache-control none --clock-control none -k regex:gft_ --csv --log-file gpurun_out/r24_steady.csv \
    python tools/r02/profile_steady.py cfg5a cfg5b rh0 > gpurun_out/r24_steady_ncu.log 2>&1
