"""Time the device-resident factorization per configuration family and break
it down per kernel class (CUDA events around every launch, separate pass).

    python tools/profile_configs.py 1:1024 2:4096 5:2048 ...
Prints one JSON line per case.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200 import configs  # noqa: E402
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device  # noqa: E402


def run(c, n, reps=int(os.environ.get("PROF_REPS", 2)), threshold=64):
    w = configs.CONFIGS[c].scaled(n)
    ctx = ffb.default_context(0)
    a0 = configs.generate_device(w, ctx)
    a = torch.empty_like(a0)
    out = DeviceBuffers(n)
    cfg = ffb.SytrfConfig(ffb.Variant.Cascade, threshold)
    st = torch.cuda.ExternalStream(ctx.stream)
    times = []
    for i in range(reps + 1):
        a.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        f = ldlt_device(a, w.p, cfg, ctx, out)
        e1.record(st)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if i > 0:
            times.append((e0.elapsed_time(e1), wall * 1e3))
    launches, syncs = ctx.launch_count(), ctx.sync_count()
    a.copy_(a0)
    torch.cuda.synchronize()
    ctx.profile(True)
    ldlt_device(a, w.p, cfg, ctx, out)
    prof = ctx.profile_read()
    ctx.profile(False)
    ms = min(t[0] for t in times)
    ops = 2.0 * n ** 3 / 3
    return dict(config=c, n=n, p=w.p, rank=f.rank, ms=ms, wall_ms=min(t[1] for t in times),
                eff_tops=ops / ms / 1e9, launches=launches, syncs=syncs,
                prof={k: dict(n=v["launches"], ms=round(v["ms"], 3),
                              tops=(v["ops"] / v["ms"] / 1e9 if v["ms"] > 0 and v["ops"] else 0))
                      for k, v in prof.items()})


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        c, n = map(int, arg.split(":"))
        try:
            print(json.dumps(run(c, n)), flush=True)
        except Exception as e:  # keep going through the list
            print(json.dumps(dict(config=c, n=n, error=str(e))), flush=True)
