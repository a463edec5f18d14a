# dense comparison GEMM after the inline-TMA / prefetch change: geometry sweep + parity tests
out=gpurun_out/r02_dense_probe2.log
: > $out
for v in "" "GFT_DG_TM=8 GFT_DG_TN=16 GFT_DG_THREADS=128" "GFT_DG_TM=8 GFT_DG_TN=8 GFT_DG_THREADS=128" "GFT_DG_TM=4 GFT_DG_TN=16" "GFT_DG_TM=2 GFT_DG_TN=16"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" >> $out 2>&1
