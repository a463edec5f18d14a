out=gpurun_out/r02_fma_probe4.log
: > $out
for v in "" "GFT_BFLY_FMA=1" "" "GFT_BFLY_FMA=1"; do
  env $v timeout 600 python tools/r02/fma_probe.py cfg5a cfg4 cfg2 cfg3 >> $out 2>&1
done
