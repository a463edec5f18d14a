"""FMA-skeleton probe: forward / inverse / fused-filter GB/s (cold burst, 20 launches) of the
configs named in argv for the kernel variant the environment selects (GFT_FMA_LOAD_PACE etc.)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

out = {"env": {k: v for k, v in os.environ.items() if k.startswith("GFT_")}}
for spec in sys.argv[1:]:
    name, dt = spec.split(":") if ":" in spec else (spec, "f32")
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=(dt,), no_cubin_cache=True)
    f = gft.Filter(p, np.exp(-p.eigenvalues()), dtypes=(dt,), no_cubin_cache=True)
    tdt = torch.float64 if dt == "f64" else torch.float32
    X = torch.randn(cfg.batch, cfg.n, device="cuda", dtype=tdt)
    Y = torch.empty_like(X)
    nb = 2 * cfg.batch * cfg.n * X.element_size()
    r = {}
    for tag, fn in (("fwd", lambda: p.forward(X, Y)), ("inv", lambda: p.inverse(X, Y)),
                    ("filt", lambda: f.apply(X, Y))):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for _rep in range(3):   # best of 3 x 60 back-to-back launches
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(60):
                fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) / 60)
        ms = best
        r[tag] = round(nb / ms / 1e6 / 6454.9, 4)
    r["kernel"] = p.kernel_name(0, dt)
    U = torch.from_numpy(p.basis()).cuda()
    Xs = X[:70001]
    p.forward(Xs, Y[:70001])
    ref = Xs.double() @ U
    r["fwd_err"] = float(((Y[:70001].double() - ref).norm(dim=1) / ref.norm(dim=1)).max())
    f.apply(Xs, Y[:70001])
    refh = ref * torch.from_numpy(np.exp(-p.eigenvalues())).cuda()
    reff = refh @ U.T
    r["filt_err"] = float(((Y[:70001].double() - reff).norm(dim=1) / reff.norm(dim=1)).max())
    out["%s_%s" % (name, dt)] = r
print(json.dumps(out))
