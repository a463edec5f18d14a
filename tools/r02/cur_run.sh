# r33: headline step A/B inside one process: FFMA2 Haar units in the tcgen05 kernels vs FADD pairs
timeout 900 python tools/r02/step_ab.py default GFT_FFMA2_UNITS=0 > gpurun_out/r33_step_ab.log 2>&1
timeout 900 python tools/r02/step_ab.py GFT_FFMA2_UNITS=0 default >> gpurun_out/r33_step_ab.log 2>&1
