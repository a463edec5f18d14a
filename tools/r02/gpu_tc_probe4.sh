GFT_TC_IOSPLIT=1 timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace_iosplit_box_hot.log 2>&1
