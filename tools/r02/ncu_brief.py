"""Key metrics of one or more ncu reports (raw page), as a markdown table on stdout."""
import csv
import io
import subprocess
import sys

M = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
     ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %"),
     ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU %"),
     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 %"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
     ("launch__registers_per_thread", "regs"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts"),
     ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
     ("smsp__inst_executed.sum", "instructions")]
print("| kernel | " + " | ".join(n for _, n in M) + " |")
print("|---|" + "---|" * len(M))
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        vals = []
        for m, _ in M:
            if m in hdr:
                i = hdr.index(m)
                vals.append("%s %s" % (r[i], units[i]) if units[i] else r[i])
            else:
                vals.append("-")
        print("| %s | %s |" % (r[hdr.index("Kernel Name")][:40], " | ".join(vals)))
