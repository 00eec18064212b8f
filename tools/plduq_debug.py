"""Small PLDUQ parity probe (parallel path forced) used for debugging on the GPU box."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1802_10453_b200 as ffb  # noqa: E402
from oracle.bind import Checker  # noqa: E402

o = Checker("oracle")
bad = 0
for p in (2, 3, 131, 8388593):
    rng = np.random.default_rng(p + 3)
    for m, n in [(1, 1), (5, 9), (64, 40), (130, 90), (300, 257), (129, 700)]:
        for kind in range(2):
            if kind == 0:
                b = rng.integers(0, p, (m, n), dtype=np.uint64)
            else:
                b = (rng.integers(0, p, (m, 2)).astype(object).dot(rng.integers(0, p, (2, n))) % p).astype(np.uint64)
            try:
                g = ffb.plduq(b, p)
            except Exception as e:
                print("EXC", p, m, n, kind, e, flush=True)
                sys.exit(1)
            r = o.plduq(p, b)
            ok = g.rank == r["rank"] and np.array_equal(g.col_perm.image_array(), r["col_image"]) \
                and np.array_equal(g.row_perm.image_array(), r["row_image"]) \
                and np.array_equal(g.lower, r["lower"]) and np.array_equal(g.upper, r["upper"])
            if not ok:
                bad += 1
                print("MISMATCH", p, m, n, kind, g.rank, r["rank"], flush=True)
print("bad", bad)
