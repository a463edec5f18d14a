# r36: warp-major tile numbering in the CUDA-core skeleton (GFT_SM_STRIPE=1): per-kernel A/B and in-step A/B
for p in cfg5a cfg4 cfg2 cfg3; do timeout 600 python tools/r02/env_confirm.py $p default GFT_SM_STRIPE=1 >> gpurun_out/r36_burst.log 2>&1; done
timeout 900 python tools/r02/step_ab.py default GFT_SM_STRIPE=1 > gpurun_out/r36_step_ab.log 2>&1
timeout 900 python tools/r02/step_ab.py GFT_SM_STRIPE=1 default >> gpurun_out/r36_step_ab.log 2>&1
