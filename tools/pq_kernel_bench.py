"""Micro-benchmark of the PLDUQ chunk kernels on synthetic inputs shaped like the
configuration-5 chunks (tools only; uses the debug export ffb_dbg_pq_bench).

    python tools/pq_kernel_bench.py            # default sweep
Row detection: S = 128 x 144 of rank k.  CRP pipeline: R_I = k x n with nz
nonzeros per row (column-sparse, like the cfg5 residual rows; rank k).
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200._lib import lib  # noqa: E402


def bench(ctx, p, which, m, reps=20):
    m = np.ascontiguousarray(m, dtype=np.uint32)
    L = lib()
    f = L.ffb_dbg_pq_bench
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                  C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    ms = (C.c_double * 3)()
    out = (C.c_int32 * (1 + 2 * max(m.shape[0], 1) + 16))()
    st = f(ctx.handle, p, which, m.shape[0], m.shape[1], m.ctypes.data, reps, ms, out)
    assert st == 0, (st, L.ffb_last_error())
    return list(ms), list(out)


def row_detect_input(rng, p, b, s, k):
    a = rng.integers(0, p, (b, k), dtype=np.int64)
    bb = rng.integers(0, p, (k, s), dtype=np.int64)
    return (a @ bb) % p


def crp_input(rng, p, k, n, nz):
    r = np.zeros((k, n), np.int64)
    for i in range(k):
        cols = rng.choice(n, nz, replace=False)
        r[i, cols] = rng.integers(1, p, nz)
    return r


def main():
    ctx = ffb.default_context(0)
    p = 131
    rng = np.random.default_rng(7)
    for k in (0, 1, 8, 25, 64, 128):
        m = row_detect_input(rng, p, 128, 144, k) if k else np.zeros((128, 144), np.int64)
        ms, out = bench(ctx, p, 0, m)
        print(json.dumps(dict(kernel="row_detect", b=128, s=144, k=k, k_found=out[0], us=round(ms[0] * 1e3, 2),
                              rrp_us=round(ms[1] * 1e3, 2), rrp_identical=bool(ms[2] == 1.0))))
    cases = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or \
        [(25, 8192, 20), (25, 8192, 400), (64, 8192, 40), (128, 16384, 100), (26, 16384, 33)]
    dump = os.environ.get("PQ_DUMP")  # an R_I written by FFB_PLDUQ_DUMP
    if dump and os.path.exists(dump):
        hdr = np.fromfile(dump, np.int64, 2)
        ri = np.fromfile(dump, np.uint32, offset=16).reshape(int(hdr[0]), int(hdr[1]))
        print("dump: k", ri.shape[0], "n", ri.shape[1], "nonzeros/row", (ri != 0).sum(1).mean(),
              "nonzero columns", int((ri != 0).any(0).sum()))
        cases = [("dump", ri)] + cases
    for case in cases:
        if case[0] == "dump":
            m = case[1]
            k, n, nz = m.shape[0], m.shape[1], -1
        else:
            k, n, nz = case
            m = crp_input(rng, p, k, n, nz)
        ms, out = bench(ctx, p, 1, m)
        print(json.dumps(dict(kernel="crp", k=k, n=n, nz=nz, fail=out[0],
                              crp_list_us=round(ms[0] * 1e3, 2), finish_us=round(ms[1] * 1e3, 2),
                              list_reg_us=round(ms[2] * 1e3, 2), list_reg_same=out[1 + 2 * k],
                              finish_phase_us=[round(x / 1e3, 2) for x in out[2 + 2 * k:7 + 2 * k]],
                              finish_reg_us=round(out[8 + 2 * k] / 1e3, 2), finish_reg_same=out[7 + 2 * k],
                              jsorted=bool(all(out[1 + i] < out[2 + i] for i in range(k - 1))))))


if __name__ == "__main__":
    main()
