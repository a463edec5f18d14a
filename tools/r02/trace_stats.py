"""Summarise a phase trace (tools/r02/trace_probe.py output): per-tile interval medians of the
last launch of CTA 0."""
import statistics
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith("TRACE cta 0")]
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 48
rows = [list(map(int, l.split(":")[1].split())) for l in lines[-nt:]]
lo, hi = 5, len(rows) - 3
names = ["load", "full", "rows", "staged", "issue", "commit", "mmadone", "drained", "outrdy", "sread",
         "st_c0", "st_c1", "st_c2", "st_c3", "af_c0", "af_c1", "af_c2", "af_c3"]
for a, b in ((0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 8), (8, 9),
             (4, 10), (10, 11), (11, 12), (12, 13), (13, 5), (2, 14), (14, 15), (15, 16), (16, 17), (17, 3)):
    x = [rows[i][b] - rows[i][a] for i in range(lo, hi)]
    print("%-8s -> %-8s median %6d min %6d max %6d" % (names[a], names[b], statistics.median(x), min(x), max(x)))
for e, nm in enumerate(names[:10]):
    x = [rows[i + 1][e] - rows[i][e] for i in range(lo, hi - 1)]
    print("period %-8s median %6d" % (nm, statistics.median(x)))
