"""Development probe of the fused C4 kernels: per-warp cycle accounting
(BTTB_FUSED_STATS=1) and per-mode CUDA-event times on the bench workload."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_06976_b200 as B  # noqa: E402
from oracle import bttb_oracle as O  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "float64"
nz = int(sys.argv[2]) if len(sys.argv) > 2 else 128
og = O.config_grid("C4", nz=nz)
g = B.make_grid(og.sx, og.sy, og.nz, 0, 0, 0, 0, og.dx, og.dy, og.z)
p = B.KernelParams.magnetic(10.0, 60.0, 50000.0)
st = B.build_transform_stack(g, p, dtype=dt)
tdt = torch.float64 if dt == "float64" else torch.float32
x = torch.rand(g.n, device="cuda", dtype=tdt) * 0.05
d = torch.randn(g.m, device="cuda", dtype=tdt)
for _ in range(3):
    y = B.apply(st, x, "forward")
    xt = B.apply(st, d, "transpose")
torch.cuda.synchronize()
for mode, v in (("forward", x), ("transpose", d)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        B.apply(st, v, mode)
    e1.record()
    torch.cuda.synchronize()
    print(f"{dt} nz={nz} {mode}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
