out=gpurun_out/r02_tc_probe5.log
: > $out
for v in "GFT_TC_IOSPLIT=1" ; do
  env $v timeout 300 python tools/r02/tc_probe.py cfg5b >> $out 2>&1
done
timeout 300 python tools/r02/tc_probe.py rh0 >> $out 2>&1
GFT_TC_IOSPLIT=1 timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace_chunk_hot.log 2>&1
timeout 300 python tools/r02/trace_probe.py rh0 3 3 > gpurun_out/r02_trace_rh0_hot.log 2>&1
