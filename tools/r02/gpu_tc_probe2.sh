out=gpurun_out/r02_tc_probe2.log
: > $out
for v in "GFT_TC_IOSPLIT=1" "GFT_TC_IOSPLIT=1 GFT_TC_PF=4" "GFT_TC_IOSPLIT=1 GFT_TC_PF=8" ""; do
  env $v timeout 300 python tools/r02/tc_probe.py cfg5b >> $out 2>&1
done
GFT_TC_IOSPLIT=1 GFT_TC_PF=4 GFT_TC_TRACE=1 timeout 300 python tools/r02/trace_probe.py cfg5b 4 > gpurun_out/r02_trace_iosplit_pf4.log 2>&1
