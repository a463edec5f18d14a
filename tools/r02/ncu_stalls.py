"""Top warp-stall reasons of each kernel in ncu reports (raw page: average warps stalled per
issue-active cycle, smsp__average_warps_issue_stalled_<reason>_per_issue_active.ratio) plus
issue-active %, as markdown.  python ncu_stalls.py report.ncu-rep ..."""
import csv
import io
import subprocess
import sys

PFX, SFX = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        st = []
        for i, h in enumerate(hdr):
            if h.startswith(PFX) and h.endswith(SFX) and "not_issued" not in h:
                try:
                    st.append((float(r[i].replace(",", "")), h[len(PFX):-len(SFX)]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        iss = r[hdr.index("smsp__issue_active.avg.pct_of_peak_sustained_active")] if \
            "smsp__issue_active.avg.pct_of_peak_sustained_active" in hdr else "?"
        print("| %s | issue active %s%% | %s |" % (name, iss, ", ".join("%s %.2f" % (n, v) for v, n in st[:6])))
