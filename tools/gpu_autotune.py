"""Offline autotuning of the FMA-skeleton geometry (rows per thread R, stages S, warps W).

Run on a B200 (under gpurun): for each (config, dtype) the fast forward kernel is JIT-built
for every candidate geometry and timed back to back (CUDA events, 30 launches); the best
geometry per (n, dtype) is written to gpurun_out/tuning.tsv, to be committed as
paper_1907_07875_b200/tuning.tsv (read by the library's choose_cfg at plan creation)."""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("cfg2", "f32"), ("cfg3", "f32"), ("cfg4", "f32"), ("cfg5a", "f32"), ("cfg4", "f64"), ("cfg1", "f32")]
# per-plan sweep (--per-plan): (config, dtype, kind); entries keyed by the kernel's leaf work
PLAN_CASES = [("cfg2", "f32", 0), ("cfg2b", "f32", 0), ("cfg3", "f32", 0), ("cfg4", "f64", 0),
              ("cfg2", "f32", 2), ("cfg3", "f32", 2), ("cfg4", "f32", 2), ("cfg4", "f64", 2),
              ("cfg5a", "f32", 2)]


def measure(cfg, dt, R, S, W, kind=0):
    env = dict(os.environ, GFT_TUNE_R=str(R), GFT_TUNE_STAGES=str(S), GFT_TUNE_WARPS=str(W), GFT_TUNING_FILE="none")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profile_kernel.py"), "--config", cfg,
                          "--dtype", dt, "--kind", str(kind), "--iters", "3"], capture_output=True, text=True,
                         env=env, timeout=300)
    for l in out.stdout.splitlines():
        if l.startswith("{"):
            return json.loads(l)
    return None


def per_plan():
    """Sweep per (config, kind, dtype); writes gpurun_out/tuning_plans.tsv with work= keys
    (work = sum k^2 of the plan for fast kernels, n^2 for the dense kernels)."""
    import workloads
    from paper_1907_07875_b200 import gft
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log = open(os.path.join(ROOT, "gpurun_out", "autotune_plans.log"), "w")
    best = {}
    for cfg, dt, kind in PLAN_CASES:
        c = workloads.config(cfg)
        plan = gft.Plan.from_config(c, dtypes=(dt,), host_only=True)
        work = c.n * c.n if kind >= 2 else plan.info()["sum_k2"]
        esz = 8 if dt == "f64" else 4
        row = c.n * esz
        for R, S, W in itertools.product((1, 2, 4, 8), (2, 3), (4, 8, 12, 16)):
            tile = 32 * R * row
            if tile < 2048 or tile > 32768 or W * S * tile > 220 * 1024:
                continue
            d = measure(cfg, dt, R, S, W, kind)
            if d is None:
                continue
            rec = {"cfg": cfg, "dtype": dt, "kind": kind, "n": c.n, "work": work, "R": R, "S": S, "W": W,
                   "b2b_ms": d["b2b_ms"], "gbs": d["b2b_gbs"]}
            log.write(json.dumps(rec) + "\n")
            log.flush()
            key = (c.n, dt, work)
            if key not in best or rec["gbs"] > best[key]["gbs"]:
                best[key] = rec
    with open(os.path.join(ROOT, "gpurun_out", "tuning_plans.tsv"), "w") as f:
        for (n, dt, work), r in sorted(best.items()):
            f.write("fma %d %s %d %d %d work=%d   # %.0f GB/s %s kind %d\n"
                    % (n, dt, r["R"], r["S"], r["W"], work, r["gbs"], r["cfg"], r["kind"]))
    print(open(os.path.join(ROOT, "gpurun_out", "tuning_plans.tsv")).read())


def main():
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log = open(os.path.join(ROOT, "gpurun_out", "autotune.log"), "w")
    best = {}
    for cfg, dt in CASES:
        import workloads
        c = workloads.config(cfg)
        esz = 8 if dt == "f64" else 4
        row = c.n * esz
        for R, S, W in itertools.product((1, 2, 4, 8), (2, 3, 4), (4, 8, 16)):
            tile = 32 * R * row
            if tile < 2048 or tile > 32768 or W * S * tile > 220 * 1024:
                continue
            d = measure(cfg, dt, R, S, W)
            if d is None:
                continue
            rec = {"cfg": cfg, "dtype": dt, "n": c.n, "R": R, "S": S, "W": W, "b2b_ms": d["b2b_ms"],
                   "gbs": d["b2b_gbs"], "grid": d["launch"]["grid"]}
            log.write(json.dumps(rec) + "\n")
            log.flush()
            best.setdefault((c.n, dt), []).append(rec)
    # per (n, dtype): the geometry with the best mean GB/s over the configs sharing the key
    chosen = {}
    for key, recs in best.items():
        cfgs = {r["cfg"] for r in recs}
        by_geo = {}
        for r in recs:
            by_geo.setdefault((r["R"], r["S"], r["W"]), {})[r["cfg"]] = r["gbs"]
        full = {g: v for g, v in by_geo.items() if set(v) == cfgs}
        g = max(full, key=lambda g: sum(full[g].values()))
        chosen[key] = {"R": g[0], "S": g[1], "W": g[2], "gbs": sum(full[g].values()) / len(cfgs),
                       "cfg": "+".join(sorted(cfgs))}
    best = chosen
    with open(os.path.join(ROOT, "gpurun_out", "tuning.tsv"), "w") as f:
        f.write("# mode n dtype R S W   (best back-to-back GB/s on B200; source config)\n")
        for (n, dt), r in sorted(best.items()):
            f.write("fma %d %s %d %d %d   # %.0f GB/s %s\n" % (n, dt, r["R"], r["S"], r["W"], r["gbs"], r["cfg"]))
    print(open(os.path.join(ROOT, "gpurun_out", "tuning.tsv")).read())


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    per_plan() if "--per-plan" in sys.argv else main()
