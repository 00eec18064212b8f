"""Measure the dense int8 tensor peak of this B200 (the roofline denominator of bench.py).

    python tools/int8_peak.py [--out gpurun_out/int8_peak.json]

Same method as the driver's MEASURED_PEAKS.json bf16 entry, for int8 -> int32:
  * library: torch._int_mm (cuBLASLt IMMA) on 8192^3, best of 10 (burst) and back to back
    for 4 s (sustained);
  * ours: the engine's persistent tcgen05 GEMM (ffb_gemm_device, C -= A*B mod 131,
    int8-centred operands, u32 C read-modify-write epilogue) on the same shape.
Ops = 2*M*N*K.  SM clocks are sampled with nvidia-smi during the sustained phase.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def clocks_during(fn):
    rows = []
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                             "--format=csv,noheader,nounits", "-lms", "100"],
                            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    th = threading.Thread(target=lambda: rows.extend(proc.stdout), daemon=True)
    th.start()
    try:
        out = fn()
    finally:
        proc.terminate()
        proc.wait(timeout=5)
        th.join(timeout=2)
    sm = [float(r.split(",")[0]) for r in rows if r.split(",")[0].strip().replace(".", "").isdigit()]
    return out, (statistics.median(sm) if sm else None)


def time_ops(call, ops, reps=10, sustain_s=4.0):
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))

    def sustained():
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.time()
        e0.record()
        while time.time() - t0 < sustain_s:
            for _ in range(8):
                call()
            n += 8
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / n

    avg, mhz = clocks_during(sustained)
    return {"burst_tops": ops / (best / 1e3) / 1e12, "burst_ms": best,
            "sustained_tops": ops / (avg / 1e3) / 1e12, "sustained_ms": avg, "sm_mhz_sustained": mhz}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "int8_peak.json"))
    ap.add_argument("--n", type=int, default=8192)
    args = ap.parse_args()
    n = args.n
    ops = 2.0 * n ** 3
    res = {"shape": [n, n, n], "how": "2*M*N*K / CUDA-event time; burst = best of 10, "
                                      "sustained = back to back for 4 s"}
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    res["torch_int_mm"] = time_ops(lambda: torch._int_mm(a, b), ops)
    del a, b
    torch.cuda.empty_cache()
    try:
        import paper_1802_10453_b200 as ffb
        from paper_1802_10453_b200._lib import lib
        from paper_1802_10453_b200.ffldl import _check
        ctx = ffb.default_context(0)
        p = 131
        A = torch.randint(0, p, (n, n), dtype=torch.int32, device="cuda")
        B = torch.randint(0, p, (n, n), dtype=torch.int32, device="cuda")
        C = torch.randint(0, p, (n, n), dtype=torch.int32, device="cuda")
        st = torch.cuda.ExternalStream(ctx.stream)
        cur = torch.cuda.current_stream()

        def call():
            # the engine runs on its own stream; join it to torch's for the events
            _check(lib().ffb_gemm_device(ctx.handle, p, 0, n, n, n, C.data_ptr(), n,
                                         A.data_ptr(), n, 0, B.data_ptr(), n, 0))
            ev = torch.cuda.Event()
            ev.record(st)
            cur.wait_event(ev)
        res["ffb_gemm_i8_tc_mod131"] = time_ops(call, ops)
    except Exception as e:  # the library peak is the point; ours is informative
        res["ffb_error"] = repr(e)
    res["int8_tops_burst"] = res["torch_int_mm"]["burst_tops"]
    res["int8_tops_sustained"] = res["torch_int_mm"]["sustained_tops"]
    res["gpu"] = torch.cuda.get_device_name(0)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
