out=gpurun_out/r02_fma_probe1.log
: > $out
for v in "" "GFT_FMA_LOAD_PACE=1"; do
  env $v timeout 600 python tools/r02/fma_probe.py cfg4 cfg4:f64 cfg5a cfg3 cfg2 >> $out 2>&1
done
