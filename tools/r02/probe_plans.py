"""Plans by short name for the r02 probes: BASELINE configs (cfg*) and the right-Haar bench
graphs (rh0 .. rh3 = workloads.RIGHT_HAAR_BENCH_CASES) and the tab:runtime graphs (tr0 .. tr6)."""
import workloads
from paper_1907_07875_b200 import gft


def make(name, batch=None, **kw):
    if name.startswith("tr"):   # workloads.tab_runtime_graphs()[I] (the paper's tab:runtime graphs)
        topo, n, build, phi, _, _ = workloads.tab_runtime_graphs()[int(name[2:])]
        s, d, w = build()
        return gft.Plan(n, s, d, w, None, phi, dtypes=("f32",), **kw), n, batch or (1 << 21), "f32"
    if name.startswith("rh"):
        case = workloads.RIGHT_HAAR_BENCH_CASES[int(name[2:])]
        n, s, d, w, loops, norm = workloads.right_haar_bench_graph(case)
        p = gft.Plan(n, s, d, w, loops, dtypes=(case[4],), normalized=norm, **kw)
        return p, n, batch or (1 << 20), case[4]
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=("f32",), **kw)
    return p, cfg.n, batch or cfg.batch, "f32"
