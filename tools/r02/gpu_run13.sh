# validation after the bench restructure + new tuning entries: bench contract test, parity of the affected
# plans (cfg1, right Haar), the driver's bench command, steady-state ncu of the rh0 kernels (DRAM % of peak)
timeout 1500 python -m pytest tests -m gpu -q -x -k "bench or right_haar or cfg1 or tune" > gpurun_out/r13_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r13_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r13_bench.log 2> gpurun_out/r13_bench.err
python tools/r02/profile_steady.py rh0 > gpurun_out/r13_steady_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --cache-control none --clock-control none -k regex:gft_ --csv --log-file gpurun_out/r13_steady_rh0.csv \
    python tools/r02/profile_steady.py rh0 cfg5b > gpurun_out/r13_steady_ncu.log 2>&1
# load-pacing optimum of the fp16x2 kernels (the sweep in r02_pace_confirm.log predates the fp16x2 split)
timeout 900 python tools/r02/pace_confirm.py rh0 1100 1150 1200 1225 1250 1275 1300 1350 > gpurun_out/r13_pace.log 2>&1
timeout 900 python tools/r02/pace_confirm.py cfg5b 2600 2650 2704 2750 2800 >> gpurun_out/r13_pace.log 2>&1
