"""Time the engine's modular GEMM on device buffers (CUDA events on the engine stream).

    python tools/gemm_bench.py [M N K] [--p 131] [--reps 5]
Prints one JSON line per shape: ms, TOPS (2MNK/t) and fraction of 4.5 POPS; also
checks one result against torch int64 arithmetic on a sample of rows.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200._lib import lib  # noqa: E402
from paper_1802_10453_b200.ffldl import _check  # noqa: E402


def run(M, N, K, p, reps, mode=0):
    ctx = ffb.default_context(0)
    st = torch.cuda.ExternalStream(ctx.stream)
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randint(0, p, (M, K), dtype=torch.int32, device="cuda", generator=g)
    B = torch.randint(0, p, (K, N), dtype=torch.int32, device="cuda", generator=g)
    C0 = torch.randint(0, p, (M, N), dtype=torch.int32, device="cuda", generator=g)
    C = C0.clone()
    torch.cuda.synchronize()
    call = lambda: _check(lib().ffb_gemm_device(ctx.handle, p, mode, M, N, K, C.data_ptr(), N,
                                                A.data_ptr(), K, 0, B.data_ptr(), N, 0))
    call()  # warm-up (+ correctness sample)
    torch.cuda.synchronize()
    rows = torch.arange(0, M, max(1, M // 7), device="cuda")[:8]
    a_s = A[rows].cpu().double()
    prod = (a_s @ B.cpu().double())  # exact: |sum| < 2^53
    ref = (C0[rows].cpu().double() - prod) % p
    ok = bool(torch.equal(ref.long(), C[rows].cpu().long()))
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        call()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ctx.profile(True)
    call()
    prof = ctx.profile_read()
    ctx.profile(False)
    ms = min(ts)
    tops = 2.0 * M * N * K / ms / 1e9
    return dict(M=M, N=N, K=K, p=p, ms=ms, tops=tops, frac_int8_peak=tops / 4500.0, correct=ok,
                kernel_ms=prof["gemm"]["ms"], pack_ms=prof["move"]["ms"],
                kernel_tops=2.0 * M * N * K / max(prof["gemm"]["ms"], 1e-9) / 1e9)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", nargs="*", type=int)
    ap.add_argument("--p", type=int, default=131)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--path", default=None, help="tc | mma | simt (FFB_GEMM_PATH)")
    a = ap.parse_args()
    if a.path:
        os.environ["FFB_GEMM_PATH"] = a.path
    shapes = [tuple(a.shape[i:i + 3]) for i in range(0, len(a.shape), 3)] or \
        [(8192, 8192, 8192), (4096, 4096, 4096), (16384, 16384, 2048), (8192, 8192, 256)]
    for s in shapes:
        r = run(*s, a.p, a.reps)
        r["path"] = a.path or "auto"
        print(json.dumps(r), flush=True)
