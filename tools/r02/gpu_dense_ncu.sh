# ncu --set full of the dense comparison GEMMs (fp32 FFMA2 4x16 tile, fp64 6x8 tile)
GFT_DG_TM=4 GFT_DG_TN=16 timeout 300 python tools/r02/dense_probe.py > gpurun_out/dn_plain1.log 2>&1 && \
GFT_DG_TM=4 GFT_DG_TN=16 ncu --set full --clock-control none --import-source on -k regex:dgfwd_f32_n128 -s 3 -c 1 -o gpurun_out/dn_f32 \
   python tools/r02/dense_probe.py > gpurun_out/dn_ncu1.log 2>&1
GFT_DG_TM=6 timeout 300 python tools/r02/dense_probe.py > gpurun_out/dn_plain2.log 2>&1 && \
GFT_DG_TM=6 ncu --set full --clock-control none --import-source on -k regex:dgfwd_f64 -s 3 -c 1 -o gpurun_out/dn_f64 \
   python tools/r02/dense_probe.py > gpurun_out/dn_ncu2.log 2>&1
