"""Summarise an FFB_PROF_TRACE file: per-class totals and GEMM time by (path, shape bucket)."""
import math
import sys
from collections import defaultdict

NAMES = ["gemm", "leaf", "rowdet", "trsm", "move", "other", "sketch", "crp", "pair", "ldu", "pack",
         "rowelim"]
recs = [l.split() for l in open(sys.argv[1])]
nodes = [int(r[5]) if len(r) > 5 else 0 for r in recs]
g = [(int(r[0]), int(r[1]), int(r[2]), int(r[3]), float(r[4])) for r in recs]
bynode = defaultdict(lambda: [0, 0.0])
for (c, m, n, k, t), nd in zip(g, nodes):
    b = 2 ** int(math.log2(max(nd, 1)))
    bynode[b][0] += 1
    bynode[b][1] += t
print("by recursion node size (launches, ms):", {k: (v[0], round(v[1], 1)) for k, v in sorted(bynode.items())})
tot = defaultdict(float)
for c, m, n, k, t in g:
    tot[NAMES[c]] += t
print({k: round(v, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1])}, round(sum(tot.values()), 1))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for c, m, n, k, t in g:
    if c != 0:
        continue
    pth = "simt" if m < 0 else ("limb" if k < 0 else ("mma" if n < 0 else "i8"))
    m, n, k = abs(m), abs(n), abs(k)
    b = lambda x: 2 ** int(math.log2(max(x, 1)))
    a = agg[(pth, b(m), b(n), b(k))]
    a[0] += 1
    a[1] += t
    a[2] += 2 * m * n * k
for key, (cnt, t, ops) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(key, cnt, round(t, 2), "ms", round(ops / t / 1e9, 1), "TOPS", round(t / cnt * 1000, 1), "us/call")

if len(sys.argv) > 3:  # TRSM breakdown: (kind, n bucket, cols bucket)
    agg = defaultdict(lambda: [0, 0.0])
    for c, m, n, k, t in g:
        if c != 3:
            continue
        b = lambda x: 2 ** int(math.log2(max(x, 1)))
        a = agg[("panel" if k == 1 else "trinv", b(m), b(n))]
        a[0] += 1
        a[1] += t
    for key, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3])]:
        print(key, cnt, round(t, 2), "ms", round(t / cnt * 1000, 1), "us/call")
