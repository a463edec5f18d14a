GFT_TC_IOSPLIT=1 GFT_TC_TRACE=1 timeout 300 python tools/r02/trace_probe.py cfg5b 4 > gpurun_out/r02_trace_iosplit.log 2>&1
GFT_TC_TRACE=1 timeout 300 python tools/r02/trace_probe.py norm32 4 > gpurun_out/r02_trace_ws32.log 2>&1 || true
