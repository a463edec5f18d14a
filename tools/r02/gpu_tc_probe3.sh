GFT_TC_IOSPLIT=1 GFT_TC_TRACE=1 timeout 300 python tools/r02/trace_probe.py cfg5b 4 > gpurun_out/r02_trace_iosplit_box.log 2>&1
cat > /tmp/one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, workloads
from paper_1907_07875_b200 import gft
cfg = workloads.config("cfg5b")
p = gft.Plan.from_config(cfg, dtypes=("f32",), no_cubin_cache=True)
X = torch.randn(cfg.batch, cfg.n, device="cuda"); Y = torch.empty_like(X)
for _ in range(4): p.forward(X, Y)
torch.cuda.synchronize()
PY
for pf in 0 4; do
GFT_TC_IOSPLIT=1 GFT_TC_PF=$pf python /tmp/one.py && GFT_TC_IOSPLIT=1 GFT_TC_PF=$pf ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum --cache-control none --clock-control none -k regex:gft_ -c 4 python /tmp/one.py > gpurun_out/r02_ncu_pf$pf.log 2>&1
done
