out=gpurun_out/r02_tc_probe8.log
: > $out
for v in "GFT_TC_N2=1" "" "GFT_TC_N2=1"; do
  env $v timeout 300 python tools/r02/tc_probe.py cfg5b >> $out 2>&1
  sleep 5
done
GFT_TC_N2=1 timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace_n2_hot.log 2>&1
