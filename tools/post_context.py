"""Which kernel precedes each read-back (k_post) in an FFB_LAUNCH_LOG stream (tools only).

    FFB_LAUNCH_LOG=1 python tools/one_factorization.py 5 32768 2> log; python tools/post_context.py log
"""
import collections
import re
import sys

names = [m.group(1) for m in (re.search(r"\] (\S+) grid", l) for l in open(sys.argv[1], errors="replace")) if m]
def demangle(n):
    m = re.search(r"(\d+)(k_\w+)", n)
    if not m:
        return n
    digits, rest = m.group(1), m.group(2)
    for d in (digits[-2:], digits[-1:]):  # the Itanium length prefix of the identifier
        L = int(d)
        if 3 <= L <= len(rest) and (L == len(rest) or rest[L] in "EI"):
            return rest[:L]
    return rest


short = [demangle(n) for n in names]
prev = collections.Counter()
seg = []
last = 0
for i, n in enumerate(short):
    if n == "k_post":
        prev[short[i - 1] if i else "-"] += 1
        seg.append(i - last)
        last = i + 1
print("launches", len(short), "posts", sum(prev.values()))
for k, v in prev.most_common(20):
    print(f"{k:28s} {v}")
hist = collections.Counter(min(s, 40) // 5 * 5 for s in seg)
pairs = collections.Counter(zip(short, short[1:]))
print("top adjacent pairs:", pairs.most_common(25))
print("launches between posts (bucket: count):", dict(sorted(hist.items())))
