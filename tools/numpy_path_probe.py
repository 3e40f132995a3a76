"""Breakdown of apply(stack, numpy, mode) on C4 (development probe): pinned
staging of the 1.03 GB model, forward, transpose."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_06976_b200 as B  # noqa: E402
from paper_1912_06976_b200 import multiply as M  # noqa: E402
from oracle import bttb_oracle as O  # noqa: E402

og = O.config_grid("C4")
g = B.make_grid(og.sx, og.sy, og.nz, 0, 0, 0, 0, og.dx, og.dy, og.z)
st = B.build_transform_stack(g, B.KernelParams.magnetic(10.0, 60.0, 50000.0))
x = np.random.default_rng(0).uniform(0, 0.05, g.n)
d = np.random.default_rng(1).normal(size=g.m)
for _ in range(2):
    B.apply(st, x, "forward"), B.apply(st, d, "transpose")


def t(f, n=3):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e3


print(f"_host_in 1.03 GB: {t(lambda: M._host_in(x, np.float64)):.1f} ms")
print(f"_host_out 1.03 GB: {t(lambda: M._host_out((g.n,), np.float64)):.1f} ms")
print(f"apply forward: {t(lambda: B.apply(st, x, 'forward')):.1f} ms")
print(f"apply transpose: {t(lambda: B.apply(st, d, 'transpose')):.1f} ms")
