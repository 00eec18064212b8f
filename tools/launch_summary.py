"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
    name = name.split("(")[0].split("<")[0].strip().split("::")[-1]
    tot[name] += v
    cnt[name] += 1
total = sum(tot.values())
print(f"launches {sum(cnt.values())}  kernel time {total / 1e3:.2f} ms (serialised, cold)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:28s} n={cnt[k]:5d}  total={v / 1e3:8.3f} ms  share={100 * v / total:5.1f}%  avg={v / cnt[k]:8.2f} us")
