"""Fused layer pipeline (csrc/pipeline.cuh, opt-in BTTB_PIPE=1) vs the oracle.

The switch is read once per process, so each case runs in a subprocess with
the environment set; the child checks parity against the CPU oracle itself.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O
dtype, layers, nb = {dtype!r}, {layers!r}, {nb!r}
og = O.config_grid("C4")
kind, consts = O.config_kernel("C4")
params = B.KernelParams.magnetic(*O.CONFIGS["C4"][11])
g = B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)
lo, hi = layers
rng = np.random.default_rng(17)
x = rng.uniform(0.0, 0.05, (2, (hi - lo) * og.n_r))
v = rng.normal(0.0, 1.0, (2, og.m))
with B.build_transform_stack(g, params, dtype=dtype, layers=layers) as st:
    f = B.apply(st, x, "forward")
    t = B.apply(st, v, "transpose")
    assert st.info()[8] >= 1
fw, tr = O.build_spectra(og, kind, consts, layers=list(range(lo, hi)))
q = (lambda a: a.astype(np.float32).astype(float)) if dtype == "float32" else (lambda a: a)
tol = 1e-10 if dtype == "float64" else 1e-5
for b in range(2):
    ef = O.rel_l2(O.forward(og, fw, q(x[b]), layers=list(range(lo, hi))), f[b])
    et = O.rel_l2(O.transpose(og, tr, q(v[b])), t[b])
    print("rel_l2", b, ef, et)
    assert ef <= tol and et <= tol, (ef, et)
print("OK")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,layers,nb", [("float64", (0, 5), 2), ("float64", (0, 5), 3),
                                             ("float32", (0, 4), 3), ("float64", (0, 1), 2)])
def test_fused_pipeline_parity(dtype, layers, nb):
    env = dict(os.environ, BTTB_PIPE="1", BTTB_PIPE_NB=str(nb))
    code = CHILD.format(root=ROOT, dtype=dtype, layers=layers, nb=nb)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
