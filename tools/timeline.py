"""Kernel timeline of one device-resident factorization (CUPTI via torch.profiler).

    python tools/timeline.py 5 32768 [out.json]

Prints, per kernel name: launches, busy ms (sum of kernel durations on the engine
stream, real run, no serialisation), and the idle gap that precedes its launches;
plus the step's span, total busy and total idle.  The gap attributed to a kernel is
the time the GPU sat idle (no kernel of ours running on any stream) just before it
started -- a read-back bubble or a launch-latency bubble.
"""
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200 import configs  # noqa: E402
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device  # noqa: E402


def main():
    c, n = int(sys.argv[1]), int(sys.argv[2])
    w = configs.CONFIGS[c].scaled(n)
    ctx = ffb.default_context(0)
    a0 = configs.generate_device(w, ctx)
    a = torch.empty_like(a0)
    out = DeviceBuffers(n)
    cfg = ffb.SytrfConfig()
    for _ in range(2):  # warm-up
        a.copy_(a0)
        torch.cuda.synchronize()
        ldlt_device(a, w.p, cfg, ctx, out)
        torch.cuda.synchronize()
    a.copy_(a0)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ldlt_device(a, w.p, cfg, ctx, out)
        torch.cuda.synchronize()
    path = sys.argv[3] if len(sys.argv) > 3 else "/tmp/ffb_timeline.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel" and e.get("ph") == "X"]
    ks = [e for e in ks if not e["name"].startswith(("at::", "void at::", "elementwise", "vectorized"))]
    ks.sort(key=lambda e: e["ts"])
    busy = defaultdict(float)
    gaps = defaultdict(float)
    cnt = defaultdict(int)
    end = ks[0]["ts"]
    idle = 0.0
    total_busy = 0.0
    for e in ks:
        mm = re.search(r"(k_\w+)", e["name"])
        nm = mm.group(1) if mm else e["name"].split("(")[0][:28]
        g = e["ts"] - end
        if g > 0:
            gaps[nm] += g
            idle += g
        cnt[nm] += 1
        busy[nm] += e["dur"]
        total_busy += max(0.0, e["ts"] + e["dur"] - max(end, e["ts"]))
        end = max(end, e["ts"] + e["dur"])
    span = end - ks[0]["ts"]
    print(f"span {span / 1e3:.2f} ms  kernels {len(ks)}  busy(union) {total_busy / 1e3:.2f} ms  "
          f"idle {idle / 1e3:.2f} ms")
    print(f"{'kernel':28s} {'n':>6s} {'busy ms':>9s} {'avg us':>8s} {'gap-before ms':>14s} {'avg gap us':>10s}")
    for nm in sorted(busy, key=lambda k: -(busy[k] + gaps[k])):
        print(f"{nm:28s} {cnt[nm]:6d} {busy[nm] / 1e3:9.3f} {busy[nm] / cnt[nm]:8.2f} "
              f"{gaps[nm] / 1e3:14.3f} {gaps[nm] / cnt[nm]:10.2f}")


if __name__ == "__main__":
    main()
