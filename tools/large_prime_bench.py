"""Large-prime contraction decision (config 3, p = 8388593 < 2^23, north star
"int8 limbs ... or an fp64 DMMA path if ncu shows it faster").

    python tools/large_prime_bench.py [--out gpurun_out/large_prime.json]

For the Schur-update shapes of config 3's recursion (n = 8192 full rank: the node of size s
updates an (s/2)^2 block with K = s/2), times with CUDA events (best of 5 after warm-up):
  * ours: ffb_gemm_device -> k_gemm_limb_tc (three signed int8 limbs, 9 tcgen05 MMAs per
    K step into 5 TMEM accumulator classes, recombined mod p in the epilogue) including
    its limb packing;
  * fp64 tensor cores: cuBLAS DGEMM (torch.matmul, float64) of the same shape -- the
    ceiling of any DMMA variant: exact for centred residues (|x| < 2^22, products < 2^44)
    only in K chunks of <= 2^9 before a reduction, which adds work on top of this time;
  * int8 reference: cuBLASLt torch._int_mm at the same shape (one int8 product).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402


def best_ms(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "large_prime.json"))
    ap.add_argument("--nodes", default="8192,4096,2048,1024", help="node sizes s (shape (s/2)^3)")
    ap.add_argument("--dgemm-only", action="store_true", help="only the cuBLAS DGEMM (ncu target)")
    args = ap.parse_args()
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200._lib import lib
    from paper_1802_10453_b200.ffldl import _check
    p = 8388593
    ctx = ffb.default_context(0)
    st = torch.cuda.ExternalStream(ctx.stream)
    rows = []
    for s in (int(x) for x in args.nodes.split(",")):
        M = N = K = s // 2
        g = torch.Generator(device="cuda").manual_seed(s)
        A = torch.randint(0, p, (M, K), dtype=torch.int32, device="cuda", generator=g)
        B = torch.randint(0, p, (K, N), dtype=torch.int32, device="cuda", generator=g)
        C0 = torch.randint(0, p, (M, N), dtype=torch.int32, device="cuda", generator=g)
        C = C0.clone()
        if args.dgemm_only:
            Ad, Bd = A.double() - p // 2, B.double() - p // 2
            for _ in range(3):
                torch.matmul(Ad, Bd)
            torch.cuda.synchronize()
            continue

        def ours():
            _check(lib().ffb_gemm_device(ctx.handle, p, 0, M, N, K, C.data_ptr(), N, A.data_ptr(), K, 0,
                                         B.data_ptr(), N, 0))
            ev = torch.cuda.Event()
            ev.record(st)
            torch.cuda.current_stream().wait_event(ev)
        C.copy_(C0)
        ours()
        torch.cuda.synchronize()
        # exactness on sampled rows (int64 on the CPU: |sum| < K p^2 < 2^59)
        idx = torch.arange(0, M, max(1, M // 5), device="cuda")[:6]
        want = (C0[idx].cpu().long() - (A[idx].cpu().long() @ B.cpu().long()) % p) % p
        ok = bool(torch.equal(want, C[idx].cpu().long()))
        t_ours = best_ms(ours)
        Ad, Bd = A.double() - p // 2, B.double() - p // 2
        t_dmma = best_ms(lambda: torch.matmul(Ad, Bd))
        Ai = torch.randint(-128, 127, (M, K), dtype=torch.int8, device="cuda")
        Bi = torch.randint(-128, 127, (K, N), dtype=torch.int8, device="cuda").t().contiguous().t()
        t_i8 = best_ms(lambda: torch._int_mm(Ai, Bi))
        ops = 2.0 * M * N * K
        row = {"node": s, "shape_mnk": [M, N, K], "exact": ok,
               "limb_tc_ms": t_ours, "limb_tc_tops": ops / t_ours / 1e9,
               "cublas_dgemm_ms": t_dmma, "cublas_dgemm_tflops": ops / t_dmma / 1e9,
               "cublaslt_int8_ms": t_i8, "cublaslt_int8_tops": ops / t_i8 / 1e9,
               "limb_vs_dgemm_speedup": t_dmma / t_ours}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del A, B, C, C0, Ad, Bd, Ai, Bi
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump({"p": p, "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
