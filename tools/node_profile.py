"""Per-launch CUDA-event profile of one factorization grouped by the size of the recursion
node each launch belongs to (FFB_PROF_TRACE; the innermost node, csrc g_node) and by kernel
class -- where the small-node launch chain spends its time.

    python tools/node_profile.py [config] [n]
"""
import os
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

CLASSES = ["gemm", "leaf", "plduq_rowdetect_seq", "trsm", "move", "other", "plduq_sketch", "plduq_crp",
           "plduq_pair", "ldu", "pack", "plduq_rowelim"]


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
    path = os.path.join(tempfile.gettempdir(), f"ffb_node_trace_{os.getpid()}.txt")
    os.environ["FFB_PROF_TRACE"] = path
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs
    from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device
    w = configs.CONFIGS[c].scaled(n)
    ctx = ffb.default_context(0)
    a0 = configs.generate_device(w, ctx)
    a = torch.empty_like(a0)
    out = DeviceBuffers(n)
    a.copy_(a0)
    ldlt_device(a, w.p, ffb.SytrfConfig(), ctx, out)
    a.copy_(a0)
    torch.cuda.synchronize()
    ctx.profile(True)
    ldlt_device(a, w.p, ffb.SytrfConfig(), ctx, out)
    ctx.profile_read()
    ctx.profile(False)
    agg = defaultdict(lambda: [0, 0.0])
    tot = defaultdict(lambda: [0, 0.0])
    shapes = defaultdict(lambda: [0, 0.0])
    for line in open(path):
        cls, m, nn, k, t, node = line.split()[:6]
        if CLASSES[int(cls)] in ("gemm", "trsm"):
            def b2(x):
                x = abs(int(x))
                return 0 if x == 0 else 1 << (x - 1).bit_length()
            shapes[(CLASSES[int(cls)], b2(m), b2(nn), b2(k))][0] += 1
            shapes[(CLASSES[int(cls)], b2(m), b2(nn), b2(k))][1] += float(t)
        b = 1 << max(0, (int(node) - 1)).bit_length()
        agg[(b, CLASSES[int(cls)])][0] += 1
        agg[(b, CLASSES[int(cls)])][1] += float(t)
        tot[b][0] += 1
        tot[b][1] += float(t)
    os.remove(path)
    print("top GEMM / TRSM shape buckets (M, N, K rounded up to powers of 2) by total ms:")
    for key, (k, t) in sorted(shapes.items(), key=lambda x: -x[1][1])[:30]:
        print(f"  {key[0]:5s} M<={key[1]:6d} N<={key[2]:6d} K<={key[3]:6d}: {k:5d} launches {t:8.3f} ms "
              f"{t / k * 1e3:7.1f} us avg")
    print(f"config {c} n={n}: launches and CUDA-event ms by node size (<= bucket) and class")
    for b in sorted(tot):
        print(f"node<={b:6d}: {tot[b][0]:6d} launches {tot[b][1]:9.3f} ms")
        for (bb, cl), (k, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            if bb == b and t > 0.05 * tot[b][1]:
                print(f"      {cl:22s} {k:6d} {t:9.3f} ms")


if __name__ == "__main__":
    main()
