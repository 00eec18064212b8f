"""Per-CUDA-source-line warp-stall samples from an ncu 'cuda,sass' source page (csv).
    ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > x.csv
    python tools/ncu_lines.py x.csv [N]
"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
path, hdr, line, src = None, None, None, {}
samp, inst, stalls = Counter(), Counter(), defaultdict(Counter)
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        line = (path, int(r[0]))
        src[line] = r[1]
    d = dict(zip(hdr[2:], r[2:]))

    def num(x):
        try:
            return int(float(x))
        except (TypeError, ValueError):
            return 0

    s = num(d.get("Warp Stall Sampling (All Samples)"))
    samp[line] += s
    inst[line] += num(d.get("Instructions Executed"))
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            stalls[line][h[6:]] += num(r[i])
tot = sum(samp.values())
print(f"total samples {tot}")
for ln, s in samp.most_common(n):
    top = ", ".join(f"{k}:{v}" for k, v in stalls[ln].most_common(3))
    print(f"{ln[0]}:{ln[1]:<5} {s:6d} ({100 * s / max(tot, 1):4.1f}%) inst={inst[ln]:7d}  [{top}]  {src.get(ln, '').strip()[:60]}")
