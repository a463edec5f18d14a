# final r02 profiles: launch list of the bench command, steady-state DRAM traffic of the headline
# kernels, ncu --set full of the dominant kernel (cfg5b forward, fp16x2 IO-split) and the rh0 kernel
python bench.py --steps 20 --warmup 5 --sustain-s 0 --cpu-budget 1 > gpurun_out/f1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f1_launches.csv \
    python bench.py --steps 20 --warmup 5 --sustain-s 0 --cpu-budget 1 > gpurun_out/f1_ncu.log 2>&1
python tools/r02/profile_steady.py > gpurun_out/f2_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
    -k regex:gft_ --csv --log-file gpurun_out/f2_steady.csv python tools/r02/profile_steady.py > gpurun_out/f2_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gft_fwdtc3s -s 2 -c 1 -o gpurun_out/f3_cfg5b_fwd \
    python tools/r02/profile_steady.py > gpurun_out/f3_ncu.log 2>&1
python tools/r02/profile_filters.py > gpurun_out/f4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gft_(fwd|filt)" -s 1 -c 100 -o gpurun_out/f4_filters \
    python tools/r02/profile_filters.py > gpurun_out/f4_ncu.log 2>&1
