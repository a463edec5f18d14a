# r67: e2e arm: equal-byte chunks per graph and the order of the graphs (fill / drain bubble)
mkdir -p gpurun_out
L=gpurun_out/r67_e2e.log; nvidia-smi --query-gpu=uuid --format=csv,noheader > $L
python tools/r02/e2e_var.py >> $L 2>&1
E2E_CHUNK_BYTES=33554432 python tools/r02/e2e_var.py >> $L 2>&1
E2E_CHUNK_BYTES=16777216 python tools/r02/e2e_var.py >> $L 2>&1
E2E_ORDER=10 python tools/r02/e2e_var.py >> $L 2>&1
E2E_CHUNK_BYTES=33554432 E2E_ORDER=10 python tools/r02/e2e_var.py >> $L 2>&1
python tools/r02/e2e_var.py >> $L 2>&1
