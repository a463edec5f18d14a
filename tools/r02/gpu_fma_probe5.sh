out=gpurun_out/r02_fma_probe5.log
: > $out
for v in "" "GFT_FMA_OBUF=1" "GFT_FMA_OBUF=2" "GFT_FMA_OBUF=1 GFT_TUNE_R=1"; do
  env $v timeout 900 python tools/r02/fma_probe.py cfg4:f64 cfg5a cfg4 cfg3 cfg2 >> $out 2>&1
done
