python tools/r02/profile_filters.py > gpurun_out/p4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gft_(fwd|filt)" -s 1 -c 100 -o gpurun_out/p4_filters \
    python tools/r02/profile_filters.py > gpurun_out/p4_ncu.log 2>&1
