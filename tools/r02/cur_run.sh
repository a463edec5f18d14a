# r57: session-5 validation at HEAD (full GPU suite, smoke, driver bench, reference arm, side tables), launch list of the
# bench command, steady-state ncu traffic of the headline + rh0 kernels, ncu --set full of the dominant kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=uuid,power.limit --format=csv,noheader > gpurun_out/r57_box.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r57_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r57_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r57_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r57_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r57_bench.log 2> gpurun_out/r57_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r57_ref.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r57_tables.json > gpurun_out/r57_bench_tables.log 2>&1
python tools/r02/profile_steady.py cfg5a cfg5b rh0 > gpurun_out/r57_steady_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --cache-control none --clock-control none -k regex:gft_ --csv --log-file gpurun_out/r57_steady.csv \
    python tools/r02/profile_steady.py cfg5a cfg5b rh0 > gpurun_out/r57_steady_ncu.log 2>&1
python bench.py --steps 20 --warmup 5 --sustain-s 0 --cpu-budget 1 > gpurun_out/r57_f1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r57_launches.csv \
    python bench.py --steps 20 --warmup 5 --sustain-s 0 --cpu-budget 1 > gpurun_out/r57_f1_ncu.log 2>&1
python tools/r02/profile_steady.py > gpurun_out/r57_f3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gft_fwdtc3s -s 2 -c 1 -o gpurun_out/r57_cfg5b_fwd \
    python tools/r02/profile_steady.py > gpurun_out/r57_f3_ncu.log 2>&1
