"""Out-of-bounds and race screens (compute-sanitizer is not
available on this GPU pool).

* Guard zones: ``tools/guard_run.py`` under BTTB_GUARD=1 -- 64 KB pattern
  zones around every library buffer and the spectrum cache, NaN canaries
  around every caller buffer, every entry point and plan family: default
  kernels, layer-chunked workspaces and the generic-length path.
* Determinism: the operator has no atomics in its reductions, so repeated
  products are bit-identical; a shared-memory or mbarrier race shows up as a
  run-to-run difference.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{}, {"BTTB_CHUNK_BYTES": "20000000"}, {"BTTB_GENERIC": "1"}],
                         ids=["default", "chunked", "generic"])
def test_guard_sweep(env):
    e = dict(os.environ, BTTB_GUARD="1", **env)
    args = [] if not env else ["small", "C1", "C4", "C5"]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "guard_run.py"), *args], env=e,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0 and "guard sweep clean" in r.stdout


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_repeated_products_bit_identical(dtype):
    og = O.config_grid("C4")
    params = B.KernelParams.magnetic(*O.CONFIGS["C4"][11])
    grid = B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)
    rng = np.random.default_rng(3)
    x = rng.uniform(0.0, 0.05, 4 * og.n_r)
    v = rng.normal(0.0, 1.0, og.m)
    with B.build_transform_stack(grid, params, dtype=dtype, layers=(60, 64)) as st:
        f0, t0 = B.apply(st, x, "forward"), B.apply(st, v, "transpose")
        for _ in range(8):
            assert np.array_equal(B.apply(st, x, "forward"), f0)
            assert np.array_equal(B.apply(st, v, "transpose"), t0)
