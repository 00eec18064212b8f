"""Micro-benchmark of the 64-row Crout leaf kernel (tools only; debug export
ffb_dbg_pq_bench, which=2): average launch time on characteristic inputs.

    python tools/leaf_bench.py [p]
zero (all pivotless), full-rank random, hollow, and L R L^T rook placements of rank
8/16/32 (the configuration-5 leaf shapes).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1802_10453_b200 as ffb  # noqa: E402
from helpers import hollow, rand_rook_rpm, rand_sym  # noqa: E402
from pq_kernel_bench import bench  # noqa: E402

if __name__ == "__main__":
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 131
    ctx = ffb.default_context(0)
    rng = np.random.default_rng(7)
    cases = {"s=1": np.ones((1, 1), np.uint64), "zero16": np.zeros((16, 16), np.uint64),
             "zero32": np.zeros((32, 32), np.uint64), "zero": np.zeros((64, 64), np.uint64),
             "full": rand_sym(rng, p, 64), "hollow": hollow(rng, p, 64)}
    for r in (8, 16, 32):
        cases[f"rook{r}"] = rand_rook_rpm(rng, p, 64, r)
    for name, a in cases.items():
        ms, out = bench(ctx, p, 2, a, reps=200)
        print(f"{name:8s} rank {out[0]:3d}  {ms[0] * 1e3:7.2f} us")
