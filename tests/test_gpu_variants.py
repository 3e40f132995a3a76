"""Parity of the library's alternative paths (environment switches, read once
per process, so each runs in its own subprocess) on the C4 geometry (2048 x
2048 FFTs), top layer block, fp64 and fp32, against the CPU oracle at the
BASELINE gates.  These are the fallbacks the default path hands over to for
other geometries (direct-read C2R, generic-team row kernels, non-TMA column
kernels, the 2000-point plan and its TMEM-free transpose), layer chunking
under a memory budget, and split launches; the default path is covered by
test_gpu_parity.py.  (The measured-slower experimental kernels of round 1
were removed: DESIGN.md section 4.)
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"float64": 1e-10, "float32": 1e-5}
LAYERS = (0, 3)
VARIANTS = ["BTTB_FWD_SPLITS=2", "BTTB_LAYER_SPLITS=4", "BTTB_QUAD=0", "BTTB_NO_TMA=1", "BTTB_FFT_POW2=0",
            "BTTB_FFT_POW2=0 BTTB_TMEM_TRA=0", "BTTB_C2R_MIRROR=0", "BTTB_T2D=0", "BTTB_CHUNK_BYTES=20000000",
            "BTTB_GENERIC=1"]

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O
og = O.config_grid("C4")
sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, dz, _, kargs, _ = O.CONFIGS["C4"]
grid = B.make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, og.z)
z = np.load({inp!r})
out = {{}}
for dt in ("float64", "float32"):
    with B.build_transform_stack(grid, B.KernelParams.magnetic(*kargs), dtype=dt, layers={layers!r}) as st:
        out["f_" + dt] = B.apply(st, z["x"], "forward")
        out["t_" + dt] = B.apply(st, z["v"], "transpose")
np.savez({outp!r}, **out)
"""


@pytest.fixture(scope="module")
def reference(tmp_path_factory):
    og = O.config_grid("C4")
    kind, consts = O.config_kernel("C4")
    lo, hi = LAYERS
    rng = np.random.default_rng(21)
    x = rng.uniform(0.0, 0.05, (hi - lo) * og.n_r)
    v = rng.uniform(0.0, 1.0, og.m)
    fw, tr = O.build_spectra(og, kind, consts, layers=list(range(lo, hi)))
    ref = {}
    for dt in ("float64", "float32"):
        xq = np.asarray(x, dtype=dt).astype(np.float64)
        vq = np.asarray(v, dtype=dt).astype(np.float64)
        ref[dt] = (O.forward(og, fw, xq, layers=list(range(lo, hi))), O.transpose(og, tr, vq))
    inp = str(tmp_path_factory.mktemp("var") / "in.npz")
    np.savez(inp, x=x, v=v)
    return inp, ref


@pytest.mark.parametrize("switch", VARIANTS)
def test_variant_parity(reference, switch, tmp_path):
    inp, ref = reference
    outp = str(tmp_path / "out.npz")
    env = dict(os.environ, **dict(kv.split("=") for kv in switch.split()))
    code = CHILD.format(root=ROOT, inp=inp, outp=outp, layers=LAYERS)
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    got = np.load(outp)
    for dt in ("float64", "float32"):
        f_ref, t_ref = ref[dt]
        assert O.rel_l2(f_ref, got["f_" + dt]) <= TOL[dt], (switch, dt, "forward")
        assert O.rel_l2(t_ref, got["t_" + dt]) <= TOL[dt], (switch, dt, "transpose")
