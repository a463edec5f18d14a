"""Wider cfg3 (n = 25 f32, odd pitch, 1-D bulk tiles) geometry sweep: fast forward and dense
forward side by side, every (R, S, W) whose SMEM fits, two repetitions (B200, under gpurun).
Output: gpurun_out/cfg3_sweep.log (one JSON line per point)."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from gpu_autotune import measure  # noqa: E402

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
log = open(os.path.join(ROOT, "gpurun_out", "cfg3_sweep.log"), "w")
row = 100
for rep in range(1):
    for R, S, W in itertools.product((1, 2, 3, 4), (2, 3, 4), (4, 5, 6, 8, 10, 12, 14, 16)):
        tile = 32 * R * row
        if W * S * tile > 224 * 1024 or tile > 16384:
            continue
        for kind in (0, 2):
            d = measure("cfg3", "f32", R, S, W, kind)
            if d is None:
                continue
            rec = {"rep": rep, "kind": kind, "R": R, "S": S, "W": W, "gbs": round(d["b2b_gbs"], 1),
                   "grid": d["launch"]["grid"]}
            log.write(json.dumps(rec) + "\n")
            log.flush()
