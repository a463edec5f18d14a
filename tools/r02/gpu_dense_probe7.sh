# dense GEMM: warps owning whole rows (no CTA barrier per tile) vs the barrier version
out=gpurun_out/r02_dense_probe7.log
: > $out
for v in "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_UNROLL=1" "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_UNROLL=4" "GFT_DG_TM=4 GFT_DG_TN=16" \
         "GFT_DG_TM=8 GFT_DG_UNROLL=4" "GFT_DG_TM=6" "GFT_DG_TM=6 GFT_DG_UNROLL=4" "GFT_DG_TM=6 GFT_DG_UNROLL=1" "GFT_DG_TM=4" \
         "GFT_DG_TM=4 GFT_DG_TN=16 GFT_DG_UNROLL=1 GFT_DG_WY=32"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
