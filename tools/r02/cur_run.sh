# r60: brute-force burst sweep of cfg5a fwd / inv geometry inside the headline step
mkdir -p gpurun_out
nvidia-smi --query-gpu=uuid --format=csv,noheader > gpurun_out/r60_fwd.log
timeout 2400 python tools/r02/step_sweep3.py fwd >> gpurun_out/r60_fwd.log 2>&1
nvidia-smi --query-gpu=uuid --format=csv,noheader > gpurun_out/r60_inv.log
timeout 2400 python tools/r02/step_sweep3.py inv >> gpurun_out/r60_inv.log 2>&1
