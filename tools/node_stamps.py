"""Phase breakdown of the fused small node k_node128 (SM-clock stamps of the last launch).
    python tools/node_stamps.py [config] [n]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200 import configs  # noqa: E402
from paper_1802_10453_b200._lib import lib  # noqa: E402
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
w = configs.CONFIGS[c].scaled(n)
ctx = ffb.default_context(0)
a0 = configs.generate_device(w, ctx)
a = torch.empty_like(a0)
out = DeviceBuffers(n)
names = ["load", "leaf(A1)", "gather B', [L1;M1]", "X = L1^-1 B'", "G = (D^-1 X)^T", "[Y;Z] update", "leaf(Z)",
         "perm + exit"]
for it in range(3):
    a.copy_(a0)
    torch.cuda.synchronize()
    ldlt_device(a, w.p, ffb.SytrfConfig(), ctx, out)
    torch.cuda.synchronize()
st = (C.c_longlong * 9)()
assert lib().ffb_dbg_node_stamps(st) == 0
d = [st[i + 1] - st[i] for i in range(8)]
print(f"config {c} n={n}: last k_node128, SM cycles (total {st[8] - st[0]})")
for nm, v in zip(names, d):
    print(f"  {nm:22s} {v:7d}")
