# confirm geometry candidates (cfg1 @ 2^24 fwd / inv / filter, right-Haar 12|20 f64); steady-state ncu of
# the rh0 kernels incl. DRAM % of peak; bench with side tables (incl. the new energy table)
out=gpurun_out/r12_confirm.log; : > $out
timeout 600 python tools/r02/geo_confirm.py cfg1@24 fwd 8,3,3,150,2 8,2,8,150,0 >> $out 2>&1
timeout 600 python tools/r02/geo_confirm.py cfg1@24 inv 8,3,3,150,2 >> $out 2>&1
timeout 600 python tools/r02/geo_confirm.py cfg1@24 filt 8,3,3,150,2 >> $out 2>&1
timeout 600 python tools/r02/geo_confirm.py rh3 fwd 1,2,1,0,0 1,2,2,0,0 >> $out 2>&1
timeout 600 python tools/r02/geo_confirm.py rh3 inv 1,2,1,0,0 1,2,2,0,0 >> $out 2>&1
python tools/r02/profile_steady.py rh0 > gpurun_out/r12_steady_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --cache-control none --clock-control none -k regex:gft_ --csv --log-file gpurun_out/r12_steady_rh0.csv \
    python tools/r02/profile_steady.py rh0 cfg5b > gpurun_out/r12_steady_ncu.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r12_tables.json > gpurun_out/r12_bench.log 2> gpurun_out/r12_bench.err
