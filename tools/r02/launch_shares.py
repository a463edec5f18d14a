"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: total device time and
launch count per kernel name, and the share of each headline-step kernel in the step."""
import csv
import io
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
start = text.index('"ID"')
tot, cnt = defaultdict(float), defaultdict(int)
first = int(sys.argv[2]) if len(sys.argv) > 2 else 100   # warm-up + timed steps: 25 x 4 launches
step_seq = []
for r in csv.DictReader(io.StringIO(text[start:])):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1.0, "us": 1e3, "ms": 1e6, "usecond": 1e3, "nsecond": 1.0, "msecond": 1e6}.get(r["Metric Unit"], 1.0)
    k = r["Kernel Name"]
    tot[k] += v * scale
    cnt[k] += 1
    if k.startswith(("gft_fwd", "gft_inv")) and len(step_seq) < first:
        step_seq.append((k, v * scale))
print("| kernel | launches | total us | mean us |")
print("|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k])[:25]:
    print("| %s | %d | %.1f | %.2f |" % (k[:60], cnt[k], tot[k] / 1e3, tot[k] / 1e3 / cnt[k]))
st, sc = defaultdict(float), defaultdict(int)
for k, v in step_seq:
    st[k] += v
    sc[k] += 1
step = {k: st[k] / sc[k] for k in st}
s = sum(step.values())
print("\nstep kernels (first %d launches = warm-up + timed steps of bench.py), mean per launch, share:" % first)
for k, v in sorted(step.items(), key=lambda kv: -kv[1]):
    print("  %s %.2f us  share %.3f" % (k, v / 1e3, v / s))
