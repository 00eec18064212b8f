"""Where the host-buffer call's time goes beyond the device-resident factorization
(tools only): pinned H2D / D2H rates, and ffb_ldlt_compact with and without the
banded upload (FFB_NO_BANDS), against ffb_ldlt_device on the same matrix.

    python tools/e2e_breakdown.py [n]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200 import configs  # noqa: E402
from paper_1802_10453_b200._lib import lib  # noqa: E402
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device  # noqa: E402
from paper_1802_10453_b200.ffldl import _check  # noqa: E402


def timed(fn, st, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    w = configs.CONFIGS[5].scaled(n)
    ctx = ffb.default_context(0)
    st = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
    a_dev = configs.generate_device(w, ctx)
    host_a = torch.empty((n, n), dtype=torch.uint8).pin_memory()
    host_a.copy_(a_dev.to(torch.uint8).cpu())
    host_l = torch.empty(n * n, dtype=torch.uint8).pin_memory()
    d8 = torch.empty((n, n), dtype=torch.uint8, device="cuda")
    res = {"n": n}
    with torch.cuda.stream(st):
        res["h2d_ms_full"] = timed(lambda: d8.copy_(host_a, non_blocking=True), st)
        res["d2h_ms_half"] = timed(lambda: host_l[: n * w.r].view(n, w.r).copy_(d8[:, : w.r], non_blocking=True), st)
    res["h2d_GBps"] = n * n / res["h2d_ms_full"] / 1e6
    del d8
    cfg = ffb.SytrfConfig()
    out = DeviceBuffers(n)
    work = torch.empty_like(a_dev)

    def dev():
        work.copy_(a_dev)
        ldlt_device(work, w.p, cfg, ctx, out)
    with torch.cuda.stream(st):
        res["device_ms"] = timed(dev, st)
    # the device run with an unrelated 1 GB H2D on a side stream at its start
    side = torch.cuda.Stream()
    d8 = torch.empty((n, n), dtype=torch.uint8, device="cuda")

    def dev_busy():
        side.wait_stream(st)
        with torch.cuda.stream(side):
            d8.copy_(host_a, non_blocking=True)
        dev()
        st.wait_stream(side)
    with torch.cuda.stream(st):
        res["device_ms_with_h2d"] = timed(dev_busy, st)
    del d8
    perm = np.zeros(n, np.int64)
    dk = np.zeros(n, np.int32)
    dv = np.zeros(n, np.uint64)
    dv2 = np.zeros(n, np.uint64)
    rank = C.c_size_t(0)
    ptr = lambda x: x.ctypes.data_as(C.c_void_p)

    def host():
        _check(lib().ffb_ldlt_compact(ctx.handle, w.p, n, host_a.data_ptr(), 1, int(cfg.variant),
                                      int(cfg.base_case_threshold), ptr(perm), host_l.data_ptr(), 1,
                                      ptr(dk), ptr(dv), ptr(dv2), C.byref(rank)))
    del a_dev, work
    for mode in ("bands", "no_bands"):
        if mode == "no_bands":
            os.environ["FFB_NO_BANDS"] = "1"
        t0 = time.perf_counter()
        res[f"e2e_ms_{mode}"] = timed(host, st)
        res[f"e2e_wall_ms_{mode}"] = (time.perf_counter() - t0) * 1e3 / 3
        os.environ.pop("FFB_NO_BANDS", None)
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
