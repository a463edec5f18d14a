timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace2_cfg5b_hot.log 2>&1
timeout 300 python tools/r02/trace_probe.py cfg5b 3 0 > gpurun_out/r02_trace2_cfg5b_cold.log 2>&1
