"""Summarise ncu captures (run here, on the CPU box) into profiles/.

  python tools/ncu_summary.py --round r01 [--dir gpurun_out]

For every gpurun_out/prof_<config>_k<kind>.ncu-rep: exports the raw page as CSV to
profiles/<round>/raw_<config>_k<kind>.csv and collects the headline metrics into
profiles/<round>/ncu_summary.md and profiles/ncu_summary.json (read by bench.py for the
roofline "traffic" field: dram read+write bytes per launch).  The launch list
(launches.csv, gpu__time_duration per launch) is copied and summarised as kernel shares.
"""
import argparse
import csv
import glob
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"0": "fast_fwd", "1": "fast_inv", "2": "dense_fwd", "3": "dense_inv"}
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "instructions"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb/issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait/issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier/issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_sb/issue"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall no_instr/issue"),
    ("launch__stack_size", "launch stack B (default 1024)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return v * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--dir", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--merge", action="store_true",
                    help="keep the rows of profiles/ncu_summary.json not re-captured this time")
    a = ap.parse_args()
    outdir = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(outdir, exist_ok=True)
    rows = []
    for rep in sorted(glob.glob(os.path.join(a.dir, "prof_*.ncu-rep"))):
        m = re.match(r"prof_(\w+?)_k(\d)(?:_(\w+))?\.ncu-rep", os.path.basename(rep))
        if not m:
            continue
        cfg, kind, tag = m.group(1), m.group(2), m.group(3)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        base = "raw_%s_k%s%s.csv" % (cfg, kind, "_" + tag if tag else "")
        with open(os.path.join(outdir, base), "w") as f:
            f.write(raw)
        r = list(csv.reader(io.StringIO(raw)))
        if len(r) < 3:
            continue
        hdr, units, vals = r[0], r[1], r[2]
        get = lambda k: (vals[hdr.index(k)], units[hdr.index(k)]) if k in hdr else (None, None)
        name = get("Kernel Name")[0]
        row = {"config": cfg, "kind": KIND[kind], "tag": tag, "kernel": name}
        for k, label in METRICS:
            v, u = get(k)
            row[label] = None if v is None else (v + (" " + u if u else ""))
        rb, ru = get("dram__bytes_read.sum")
        wb, wu = get("dram__bytes_write.sum")
        if rb is not None:
            row["dram_bytes_per_launch"] = to_bytes(rb, ru) + to_bytes(wb, wu)
        rows.append(row)
    if a.merge:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            old_rows = json.load(f)["kernels"]
        fresh = {(r["config"], r["kind"], r["tag"]) for r in rows}
        rows = [r for r in old_rows if (r["config"], r["kind"], r["tag"]) not in fresh] + rows
        order = ["cfg1big", "cfg2", "cfg2b", "cfg3", "cfg4", "cfg5a", "cfg5b"]
        rows.sort(key=lambda r: (order.index(r["config"]) if r["config"] in order else 99, r["kind"],
                                 r["tag"] or ""))
    # launch list
    shares = {}
    lc = os.path.join(a.dir, "launches.csv")
    if os.path.exists(lc):
        with open(lc) as f:
            text = f.read()
        with open(os.path.join(outdir, "launches.csv"), "w") as f:
            f.write(text)
        lines = [l for l in text.splitlines() if l.startswith('"')]
        rd = list(csv.reader(io.StringIO("\n".join(lines))))
        if rd:
            h = rd[0]
            for rr in rd[1:]:
                if rr[h.index("Metric Name")] != "gpu__time_duration.sum":
                    continue
                nm = rr[h.index("Kernel Name")]
                key = re.sub(r"_[0-9a-f]{16}$", "", nm)
                shares[key] = shares.get(key, 0.0) + float(rr[h.index("Metric Value")].replace(",", ""))
    tot = sum(shares.values()) or 1.0
    with open(os.path.join(outdir, "ncu_summary.md"), "w") as f:
        f.write("# ncu summary (%s)\n\nSource: `ncu --set full --clock-control none` captures of "
                "`tools/profile_kernel.py` (one launch, cold cache, serialised).  Durations under ncu are "
                "not bench numbers.\n\n" % a.round)
        labels = ["config", "kind", "tag"] + [l for _, l in METRICS] + ["dram_bytes_per_launch"]
        f.write("| " + " | ".join(labels) + " |\n|" + "---|" * len(labels) + "\n")
        for r in rows:
            f.write("| " + " | ".join(str(r.get(l)) for l in labels) + " |\n")
        if shares:
            f.write("\n## Launch list shares (bench.py run under `ncu --metrics gpu__time_duration.sum`)\n\n")
            f.write("| kernel | total ns | share |\n|---|---|---|\n")
            for k, v in sorted(shares.items(), key=lambda kv: -kv[1]):
                f.write("| %s | %.0f | %.3f |\n" % (k, v, v / tot))
            # the bench step is the fast forward + fast inverse; the dense (gft_d*) comparison
            # kernels run after the timed region
            step = {k: v for k, v in shares.items() if re.match(r"gft_(fwd|inv)", k)}
            st = sum(step.values()) or 1.0
            f.write("\nShare of the bench step (fast forward + fast inverse only; the dense `gft_d*` "
                    "kernels are the comparison timed after the step): " +
                    ", ".join("%s %.3f" % (k, v / st) for k, v in sorted(step.items())) + ".\n")
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump({"round": a.round, "kernels": rows, "launch_shares": {k: v / tot for k, v in shares.items()}},
                  f, indent=1)
    # multi-kernel capture of tools/profile_many.py (right Haar / approximate rows): every
    # kernel is launched twice, the second (warm-module) launch of each spec is reported
    rep = os.path.join(a.dir, "prof_next_rows.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(outdir, "raw_next_rows.csv"), "w") as f:
            f.write(raw)
        r = list(csv.reader(io.StringIO(raw)))
        specs = []
        pm = os.path.join(a.dir, "plain_many.log")
        if os.path.exists(pm):
            for line in open(pm):
                try:
                    v = json.loads(line)
                except ValueError:
                    continue
                specs.extend(v if isinstance(v, list) else [v])
        if len(r) >= 3:
            hdr, units = r[0], r[1]
            cols = [("Kernel Name", "kernel")] + METRICS[:11]
            with open(os.path.join(outdir, "ncu_next_rows.md"), "w") as f:
                f.write("# ncu --set full: right Haar / approximate kernels (%s)\n\nSource: `ncu --set full "
                        "--clock-control none -k regex:gft_` of `tools/profile_many.py` (each kernel launched "
                        "twice, cold, serialised; the second launch is listed).  Raw page: `raw_next_rows.csv`.  "
                        "Durations under ncu are not bench numbers.\n\n" % a.round)
                f.write("| spec | " + " | ".join(l for _, l in cols) + " |\n|" + "---|" * (len(cols) + 1) + "\n")
                for i, vals in enumerate(r[2:]):
                    if i % 2 == 0:
                        continue
                    spec = specs[i // 2].get("spec", "") if i // 2 < len(specs) else ""
                    cells = []
                    for k, _ in cols:
                        j = hdr.index(k) if k in hdr else -1
                        cells.append("" if j < 0 else vals[j] + ((" " + units[j]) if units[j] else ""))
                    f.write("| %s | %s |\n" % (spec, " | ".join(cells)))
    print("wrote", outdir)


if __name__ == "__main__":
    main()
