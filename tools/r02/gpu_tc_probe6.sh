out=gpurun_out/r02_tc_probe6.log
: > $out
for v in "GFT_TC_IOSPLIT=1" "" "GFT_TC_SPLIT=rna"; do
  env $v timeout 300 python tools/r02/tc_probe.py cfg5b >> $out 2>&1
  sleep 5
done
timeout 300 python tools/r02/tc_probe.py rh0 >> $out 2>&1
