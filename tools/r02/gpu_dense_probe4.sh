# FFMA2 dense GEMM vs scalar FFMA, fp64 6-row tiles
out=gpurun_out/r02_dense_probe4.log
: > $out
python tools/r02/peaks_probe.py >> $out 2>&1
for v in "" "GFT_DG_FFMA2=0" "GFT_DG_TM=6" "GFT_DG_TM=16 GFT_DG_THREADS=128" "GFT_DG_TM=4 GFT_DG_TN=16" "GFT_DG_TM=8 GFT_DG_TN=16 GFT_DG_THREADS=128"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
python tools/r02/peaks_probe.py >> $out 2>&1
