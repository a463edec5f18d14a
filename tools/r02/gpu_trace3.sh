timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace3_base_hot.log 2>&1
GFT_TC_EXP_NOSTTM=1 timeout 300 python tools/r02/trace_probe.py cfg5b 3 3 > gpurun_out/r02_trace3_nosttm_hot.log 2>&1
GFT_TC_EXP_NOSTTM=1 timeout 300 python tools/r02/tc_probe.py cfg5b 2 > gpurun_out/r02_tc_nosttm.log 2>&1
