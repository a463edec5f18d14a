out=gpurun_out/r02_tc_probe1.log
: > $out
for v in "GFT_TC_SPLIT=rna" "" "GFT_TC_IOSPLIT=1" "GFT_TC_SPLIT=rna GFT_TC_IOSPLIT=1"; do
  env $v timeout 300 python tools/r02/tc_probe.py cfg5b >> $out 2>&1
done
