# r42: re-entry validation at HEAD (full GPU suite, smoke, driver bench, reference arm), launch list of the bench command,
# steady-state ncu traffic of the headline + rh0 kernels, ncu --set full of the dominant kernel
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r42_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r42_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r42_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r42_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r42_bench.log 2> gpurun_out/r42_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r42_ref.log 2>&1
python tools/r02/profile_steady.py cfg5a cfg5b rh0 > gpurun_out/r42_steady_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --cache-control none --clock-control none -k regex:gft_ --csv --log-file gpurun_out/r42_steady.csv \
    python tools/r02/profile_steady.py cfg5a cfg5b rh0 > gpurun_out/r42_steady_ncu.log 2>&1
python bench.py --steps 20 --warmup 5 --sustain-s 0 --cpu-budget 1 > gpurun_out/r42_f1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r42_launches.csv \
    python bench.py --steps 20 --warmup 5 --sustain-s 0 --cpu-budget 1 > gpurun_out/r42_f1_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gft_invtc3s -s 2 -c 1 -o gpurun_out/r42_cfg5b_inv \
    python tools/r02/profile_steady.py > gpurun_out/r42_f3_ncu.log 2>&1
