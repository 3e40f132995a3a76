"""One small operator case for compute-sanitizer (tools/sanitize.sh).

usage: python tools/sanitize_case.py {C1,C2,C4L} [float64|float32]
C1 / C2: the BASELINE gravity / magnetic 50x40x10 configs; C4L: the C4
geometry (1000 x 1000 stations, 2048 x 2048 FFTs) on a two-layer block.
Runs forward + transpose through the C ABI and checks the oracle gate, so a
sanitizer run also proves the instrumented run computed the right answer.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1912_06976_b200 as B  # noqa: E402
from oracle import bttb_oracle as O  # noqa: E402

name = sys.argv[1]
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
tol = 1e-10 if dtype == "float64" else 1e-5
cfg = "C4" if name == "C4L" else name
og = O.config_grid(cfg)
kind, consts = O.config_kernel(cfg)
params = B.KernelParams.gravity() if kind == "gravity" else B.KernelParams.magnetic(*O.CONFIGS[cfg][11])
layers = (0, 2) if name == "C4L" else (0, og.nz)
lo, hi = layers
rng = np.random.default_rng(5)
x = rng.uniform(0.0, 0.05, (hi - lo) * og.n_r)
v = rng.uniform(0.0, 1.0, og.m)
grid = B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)
with B.build_transform_stack(grid, params, dtype=dtype, layers=layers) as st:
    f = B.apply(st, x, "forward")
    t = B.apply(st, v, "transpose")
fw, tr = O.build_spectra(og, kind, consts, layers=list(range(lo, hi)))
q = lambda a: np.asarray(a, dtype=dtype).astype(np.float64)  # noqa: E731
ef = O.rel_l2(O.forward(og, fw, q(x), layers=list(range(lo, hi))), f)
et = O.rel_l2(O.transpose(og, tr, q(v)), t)
print(f"{name} {dtype} pipe={os.environ.get('BTTB_PIPE', '0')}: forward {ef:.2e} transpose {et:.2e}")
sys.exit(0 if ef <= tol and et <= tol else 1)
