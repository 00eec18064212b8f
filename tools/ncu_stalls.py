"""Warp-state totals of one kernel from an ncu report captured with --import-source on
(--warp-sampling-interval 0 for short kernels): duration, instructions, stall reasons summed
over all source lines, then the hottest lines (tools/ncu_lines.py).
    python tools/ncu_stalls.py rep.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, rx = sys.argv[1], sys.argv[2]
top = sys.argv[3] if len(sys.argv) > 3 else "25"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{rx}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
print(f"# {rep}  kernel {v[h.index('Kernel Name')][:60]}  grid {v[h.index('Grid Size')]} block {v[h.index('Block Size')]}")
for k in ("gpu__time_duration.sum", "sm__cycles_active.max", "smsp__inst_executed.sum", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum"):
    if k in h:
        print(f"{k}: {v[h.index(k)]} {rows[1][h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{rx}"],
                     capture_output=True, text=True).stdout
open("/tmp/_ncu_src.csv", "w").write(src)
hdr, tot = None, Counter()
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    for i, x in enumerate(hdr):
        if x.startswith("stall_") and "Not Issued" not in x:
            try:
                tot[x[6:]] += int(float(r[i]))
            except ValueError:
                pass
s = sum(tot.values()) or 1
print("warp-state samples (all lines):", ", ".join(f"{k} {100 * n / s:.1f}%" for k, n in tot.most_common(8)))
print(subprocess.run([sys.executable, __file__.replace("ncu_stalls.py", "ncu_lines.py"), "/tmp/_ncu_src.csv", top],
                     capture_output=True, text=True).stdout)
