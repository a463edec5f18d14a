out=gpurun_out/r02_f16_probe.log
: > $out
GFT_TC_F16=1 timeout 300 python tools/r02/tc_probe.py cfg5b 2 >> $out 2>&1
sleep 5
timeout 300 python tools/r02/tc_probe.py cfg5b 2 >> $out 2>&1
sleep 5
GFT_TC_F16=1 timeout 300 python tools/r02/tc_probe.py rh1 2 >> $out 2>&1
GFT_TC_F16=1 timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace_f16_hot.log 2>&1
