"""One-screen summary of the first kernel of an ncu report (details page + the tensor-pipe,
DRAM and SM counters bench/DESIGN quote).  python tools/ncu_summary.py rep.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
keep = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Memory Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "SM Frequency",
        "L2 Hit Rate")
print(f"# {title}")
seen = set()
name = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("ID") != "0":
        continue
    name = d.get("Kernel Name", name)
    n = d.get("Metric Name", "")
    if n in keep and n not in seen:
        seen.add(n)
        print(f"{n}: {d.get('Metric Value')} {d.get('Metric Unit')}")
print(f"kernel: {(name or '')[:100]}")
rr = list(csv.reader(io.StringIO(raw)))
h, u, v = rr[0], rr[1], rr[2]
for key in ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
            "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
    for i, name in enumerate(h):  # section-prefixed names (e.g. TPC.TriageCompute.<metric>)
        if name == key or name.endswith("." + key):
            print(f"{key}: {v[i]} {u[i]}")
            break
