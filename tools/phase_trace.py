"""Phase timeline of the large nodes of one factorization (FFB_PHASE_TRACE event marks,
no synchronisation inside the run).   python tools/phase_trace.py 5 32768 [min_node]"""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.join(tempfile.gettempdir(), f"ffb_phase_{os.getpid()}.txt")
os.environ["FFB_PHASE_TRACE"] = path
if len(sys.argv) > 3:
    os.environ["FFB_PHASE_MIN"] = sys.argv[3]
import torch  # noqa: E402

import paper_1802_10453_b200 as ffb  # noqa: E402
from paper_1802_10453_b200 import configs  # noqa: E402
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device  # noqa: E402

c, n = int(sys.argv[1]), int(sys.argv[2])
w = configs.CONFIGS[c].scaled(n)
ctx = ffb.default_context(0)
a0 = configs.generate_device(w, ctx)
a = torch.empty_like(a0)
out = DeviceBuffers(n)
for _ in range(3):
    a.copy_(a0)
    torch.cuda.synchronize()
    if os.path.exists(path):
        os.remove(path)
    ldlt_device(a, w.p, ffb.SytrfConfig(), ctx, out)
    torch.cuda.synchronize()
print(open(path).read())
