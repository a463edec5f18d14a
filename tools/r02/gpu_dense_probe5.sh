# dense GEMM: tile x unroll x software prefetch with FFMA2
out=gpurun_out/r02_dense_probe5.log
: > $out
for v in "GFT_DG_TM=8" "GFT_DG_TM=4 GFT_DG_TN=16" "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_UNROLL=4" "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_UNROLL=1" \
         "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_PREFETCH=1" "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_PREFETCH=1 GFT_DG_UNROLL=4" \
         "GFT_DG_TM=8 GFT_DG_UNROLL=4" "GFT_DG_TM=8 GFT_DG_PREFETCH=1" \
         "GFT_DG_TM=6 GFT_DG_UNROLL=4" "GFT_DG_TM=6 GFT_DG_PREFETCH=1" "GFT_DG_TM=6 GFT_DG_UNROLL=1" "GFT_DG_TM=2 GFT_DG_TN=16" "GFT_DG_TM=6 GFT_DG_TN=16"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
