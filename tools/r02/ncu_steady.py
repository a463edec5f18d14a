"""Parse `ncu --csv` output of tools/r02/profile_steady.py (metrics dram__bytes_read.sum,
dram__bytes_write.sum, gpu__time_duration.sum) into profiles/ncu_steady.json: per kernel name
the mean DRAM bytes per launch over launches 2..N (steady state) and the first launch's."""
import csv
import io
import json
import statistics
import sys
from collections import defaultdict

rows = defaultdict(lambda: defaultdict(list))
text = open(sys.argv[1]).read()
start = text.index('"ID"')
for r in csv.DictReader(io.StringIO(text[start:])):
    k = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)
    rows[k][r["Metric Name"]].append(v * scale)
out = {"how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "--cache-control none --clock-control none of tools/r02/profile_steady.py (6 back-to-back "
              "launches per kernel); steady state = mean of launches 2..6",
       "kernels": {}}
for k, m in rows.items():
    rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    out["kernels"][k] = {"launches": len(rd),
                         "dram_bytes_per_launch": round(statistics.mean([a + b for a, b in zip(rd[1:], wr[1:])])),
                         "dram_read_per_launch": round(statistics.mean(rd[1:])),
                         "dram_write_per_launch": round(statistics.mean(wr[1:])),
                         "first_launch_bytes": round(rd[0] + wr[0]),
                         "duration_us_mean": round(statistics.mean(m["gpu__time_duration.sum"][1:]), 2)}
    pct = m.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    if pct:
        out["kernels"][k]["dram_pct_of_peak_mean"] = round(statistics.mean(pct[1:]), 2)
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
