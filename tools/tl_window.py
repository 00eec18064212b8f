"""Kernels of a tools/timeline.py trace inside a time window, one line per kernel:
start (us from the first kernel), duration, stream, name.
    python tools/tl_window.py trace.json[.gz] t0_ms t1_ms"""
import gzip
import json
import re
import sys

path, t0, t1 = sys.argv[1], float(sys.argv[2]) * 1e3, float(sys.argv[3]) * 1e3
ev = json.load(gzip.open(path) if path.endswith(".gz") else open(path))["traceEvents"]
ks = [e for e in ev if e.get("cat") == "kernel" and e.get("ph") == "X"]
ks.sort(key=lambda e: e["ts"])
z = ks[0]["ts"]
streams = {}
for e in ks:
    s = e["args"].get("stream")
    streams.setdefault(s, len(streams))
    a = e["ts"] - z
    if a + e["dur"] < t0 or a > t1:
        continue
    nm = (re.search(r"(k_\w+)", e["name"]) or re.search(r"(\w+)", e["name"])).group(1)
    g = e["args"].get("grid", "")
    print(f"{a:10.1f} {e['dur']:8.1f}  s{streams[s]}  {nm:24s} {g}")
