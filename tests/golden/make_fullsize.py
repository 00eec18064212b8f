"""Generate tests/golden/fullsize.json -- SHA-256 digests of the oracle's (P, L, D, rank)
for the five BASELINE.json configurations at their stated sizes.

TEST INFRASTRUCTURE ONLY.  The CPU oracle (oracle/ldlt_oracle.c, itself pinned against the
unmodified reference in tests/test_oracle.py) factors the seeded config inputs
(csrc/ffb_gen.cu host generator, bit-identical to the device generator) with the
reference's default {Cascade, 64} (sytrf.hpp:14-17).  The GPU test
tests/test_fullsize_gpu.py::test_full_size_bit_exact hashes ffb_ldlt_device's outputs the
same way and compares.  With --ref, a configuration is also factored by the UNMODIFIED
reference (oracle/_ref) and the digests must agree (cfg2: ~250 s single-threaded).

Digest layout (all little-endian):
  perm   int64[n]            image(pos) = original row (permutation.hpp:11-19)
  lower  uint32[n, r]        row-major, in blocks of BLOCK rows (one digest per block)
  dkind  int32[r]            0 Scalar, 1/2 AntiDiag, 3/4 AntiTri (blockdiag.hpp:20-33)
  dval   uint32[r], dval2 uint32[r]

Usage: python tests/golden/make_fullsize.py [--configs 1,2,3,4,5] [--ref 1,2]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT = os.path.join(HERE, "fullsize.json")
BLOCK = 4096


def _h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def digest(perm, lower, dkind, dval, dval2, rank: int) -> dict:
    """perm/lower/... as numpy arrays (lower: n x >=rank, any integer dtype)."""
    n = perm.shape[0]
    blocks = []
    for r0 in range(0, n, BLOCK):
        blk = np.ascontiguousarray(lower[r0:r0 + BLOCK, :rank]).astype(np.uint32, copy=False)
        blocks.append(_h(blk))
    return {
        "rank": int(rank),
        "perm": _h(np.asarray(perm, np.int64)),
        "lower_blocks": blocks,
        "dkind": _h(np.asarray(dkind[:rank], np.int32)),
        "dval": _h(np.asarray(dval[:rank], np.uint32)),
        "dval2": _h(np.asarray(dval2[:rank], np.uint32)),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--ref", default="", help="configs also run through the unmodified reference")
    args = ap.parse_args()
    from oracle.bind import Checker
    from paper_1802_10453_b200 import configs

    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data.setdefault("_about", "SHA-256 digests of the CPU oracle's P, L, D, rank at BASELINE.json "
                              "sizes; made by tests/golden/make_fullsize.py")
    data["_block_rows"] = BLOCK
    oracle = Checker("oracle")
    ref_set = {int(c) for c in args.ref.split(",") if c}
    for c in (int(x) for x in args.configs.split(",")):
        w = configs.CONFIGS[c]
        a = configs.generate(w)
        t0 = time.time()
        o = oracle.ldlt(w.p, a, "cascade", 64)
        dt = time.time() - t0
        d = digest(o.perm, o.lower, o.dkind, o.dval, o.dval2, o.rank)
        d.update(n=w.n, p=w.p, seed=w.seed, rank_param=w.r, oracle_s=round(dt, 1),
                 variant="cascade", threshold=64)
        print(f"config {c}: n={w.n} rank={o.rank} oracle {dt:.1f} s", flush=True)
        del o
        if c in ref_set:
            t0 = time.time()
            r = Checker("ref").ldlt(w.p, a, "cascade", 64)
            rt = time.time() - t0
            dr = digest(r.perm, r.lower, r.dkind, r.dval, r.dval2, r.rank)
            same = all(dr[k] == d[k] for k in ("rank", "perm", "lower_blocks", "dkind", "dval", "dval2"))
            print(f"config {c}: unmodified reference {rt:.1f} s, digests equal: {same}", flush=True)
            if not same:
                raise SystemExit(f"config {c}: oracle and unmodified reference differ")
            d["reference_checked"] = True
            d["reference_s"] = round(rt, 1)
        elif data.get(str(c), {}).get("reference_checked") and data[str(c)].get("perm") == d["perm"]:
            d["reference_checked"] = True
            d["reference_s"] = data[str(c)].get("reference_s")
        data[str(c)] = d
        del a
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
