"""Back-to-back launches for the steady-state ncu traffic capture: each of the headline
workload's four kernels (cfg5a / cfg5b forward and inverse) launched 6 times in a row on
device-resident inputs > L2.  Under `ncu --cache-control none` the dirty L2 lines one launch
leaves behind are written back during the next, so the mean DRAM bytes of launches 2..6 is
the steady-state traffic per launch (a single cold launch under-counts writes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import probe_plans  # noqa: E402

# plans by probe name (default: the headline's cfg5a and cfg5b; e.g. rh0 for the right-Haar 32|32 kernel)
for name in (sys.argv[1:] or ["cfg5a", "cfg5b"]):
    p, n, batch, dt = probe_plans.make(name)
    X = torch.randn(batch, n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
    Y = torch.empty_like(X)
    for kind, f in ((0, p.forward), (1, p.inverse)):
        print(name, kind, p.kernel_name(kind, dt), flush=True)
        for _ in range(6):
            f(X, Y)
        torch.cuda.synchronize()
