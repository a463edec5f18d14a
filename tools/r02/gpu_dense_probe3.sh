out=gpurun_out/r02_dense_probe3.log
: > $out
python tools/r02/peaks_probe.py >> $out 2>&1
for v in "" "GFT_DG_PREFETCH=1" "GFT_DG_TM=8 GFT_DG_TN=8 GFT_DG_THREADS=128" ; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
