"""Critical-path attribution of a tools/timeline.py trace: each kernel is charged
the time from max(previous end, its start) to its end (PDL pre-launch waits are
not charged).  python tools/tl_attr.py trace.json[.gz] [top]"""
import gzip
import json
import re
import sys
from collections import defaultdict

path = sys.argv[1]
ev = json.load(gzip.open(path) if path.endswith(".gz") else open(path))["traceEvents"]
ks = [e for e in ev if e.get("cat") == "kernel" and e.get("ph") == "X"]
ks.sort(key=lambda e: e["ts"] + e["dur"])
nm = lambda s: (re.search(r"(k_\w+)", s) or re.search(r"(\w+)", s)).group(1)
eff, cnt = defaultdict(float), defaultdict(int)
end = ks[0]["ts"]
for e in ks:
    t_end = e["ts"] + e["dur"]
    eff[nm(e["name"])] += max(0.0, t_end - max(end, e["ts"]))
    cnt[nm(e["name"])] += 1
    end = max(end, t_end)
tot = sum(eff.values())
print(f"span {(end - ks[0]['ts']) / 1e3:.2f} ms, {len(ks)} kernels")
for k in sorted(eff, key=lambda k: -eff[k])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"  {k:26s} {cnt[k]:6d} {eff[k] / 1e3:8.3f} ms {eff[k] / cnt[k]:7.2f} us {100 * eff[k] / tot:5.1f}%")
