import sys, os
sys.path.insert(0, '/root/repo')
import paper_1802_10453_b200 as ffb
from paper_1802_10453_b200 import configs
from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device
import torch
w = configs.CONFIGS[5].scaled(256)
ctx = ffb.default_context(0)
a = configs.generate_device(w, ctx)
out = DeviceBuffers(256)
f = ldlt_device(a, w.p, ffb.SytrfConfig(ffb.Variant.Cascade, 64), ctx, out)
print("rank", f.rank, "launches", ctx.launch_count(), "syncs", ctx.sync_count())
