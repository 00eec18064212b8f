"""One device-resident factorization of a configuration-family matrix (tools only;
the program an ncu launch list is taken of).

    python tools/one_factorization.py 5 32768
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200 import configs  # noqa: E402
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device  # noqa: E402

c, n = int(sys.argv[1]), int(sys.argv[2])
w = configs.CONFIGS[c].scaled(n)
ctx = ffb.default_context(0)
a = configs.generate_device(w, ctx)
f = ldlt_device(a, w.p, ffb.SytrfConfig(), ctx, DeviceBuffers(n))
torch.cuda.synchronize()
print("rank", f.rank, "expected", w.r)
