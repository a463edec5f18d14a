out=gpurun_out/r02_fma_probe2.log
: > $out
for v in "" "GFT_TUNE_WARPS=6" "GFT_TUNE_WARPS=7" "GFT_TUNE_WARPS=6 GFT_TUNE_STAGES=2 GFT_TUNE_R=1"; do
  env $v timeout 600 python tools/r02/fma_probe.py cfg4:f64 >> $out 2>&1
done
for v in "" "GFT_TUNE_WARPS=12" "GFT_TUNE_WARPS=10" "GFT_TUNE_WARPS=12 GFT_TUNE_STAGES=2 GFT_TUNE_R=1"; do
  env $v timeout 600 python tools/r02/fma_probe.py cfg5a >> $out 2>&1
done
