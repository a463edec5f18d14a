# dense comparison GEMM geometry sweep (tools/r02/dense_probe.py) + ncu of the default cfg5b kernel
out=gpurun_out/r02_dense_probe.log
: > $out
for v in "" "GFT_DG_TM=4 GFT_DG_TN=16" "GFT_DG_TM=8 GFT_DG_TN=16 GFT_DG_THREADS=128" "GFT_DG_TM=16 GFT_DG_TN=8 GFT_DG_THREADS=128" "GFT_DG_TM=4 GFT_DG_TN=8" "GFT_DG_TM=8 GFT_DG_TN=4"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
cat > /tmp/dprof.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, workloads
from paper_1907_07875_b200 import gft
for name, dt in (("cfg5b", "f32"), ("cfg4", "f64")):
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=(dt,))
    X = torch.randn(cfg.batch, cfg.n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
    Y = torch.empty_like(X)
    p.dense_forward(X, Y); p.dense_forward(X, Y)
    torch.cuda.synchronize()
PY
python /tmp/dprof.py && ncu --set full --clock-control none --import-source on -k regex:gft_dg -c 4 -o gpurun_out/r02_dense_prof python /tmp/dprof.py > gpurun_out/r02_dense_ncu.log 2>&1
