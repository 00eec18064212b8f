"""Summarise an ncu SASS source page (csv on stdin): the hottest instructions by
warp-stall samples and by executed instructions.  Usage:
    ncu -i rep --page source --csv --print-source sass -k regex:NAME | python tools/ncu_hot.py [N]
"""
import csv
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25
rows = list(csv.reader(sys.stdin))
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
ins = sum(int(d["Instructions Executed"] or 0) for d in data)
print(f"samples={tot} warp_instructions={ins} sass_lines={len(data)}")
for i, d in enumerate(data):
    d["_i"] = i
hot = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:n]
for d in sorted(hot, key=lambda d: d["_i"]):
    print(f'{d["_i"]:5d} {d["Warp Stall Sampling (All Samples)"]:>6} {d["Instructions Executed"]:>8}  {d["Source"].strip()[:70]}')
