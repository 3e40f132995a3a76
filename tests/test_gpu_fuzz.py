"""Seeded geometry sweep of the sm_100a operator against the CPU oracle.

The BASELINE configs exercise a handful of FFT lengths; this sweep draws
random station grids, paddings (including one-sided and zero), layer counts,
cell sizes and uneven depth blocks, so that every FFT length family the plan
can pick (2^a, 2^a 3^b, 2^a 5^b; compile-time and runtime-radix plans), odd
and even embeddings and ragged last row pairs / column teams are covered.
Gates: relative L2 <= 1e-10 (fp64) and <= 1e-5 (fp32), forward and transpose,
gravity and magnetic (BASELINE.json north_star).  Edge cases the reference
tests hold: one station row or column (sx = 1 / sy = 1), one layer, a single
prism.
"""
import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-10, "float32": 1e-5}


def draw(seed):
    rng = np.random.default_rng(seed)
    sx, sy = (int(v) for v in rng.integers(1, 140 if seed % 4 == 0 else 70, 2))
    pads = [int(v) for v in rng.integers(0, 6, 4)]
    if seed % 3 == 0:
        pads = [pads[0], 0, 0, pads[3]]  # one-sided padding
    nz = int(rng.integers(1, 5))
    dx, dy = (float(v) for v in rng.uniform(5.0, 80.0, 2))
    z = np.concatenate([[0.0], np.cumsum(rng.uniform(3.0, 60.0, nz))])
    return sx, sy, nz, pads, dx, dy, z


CASES = [(s, k) for s in range(40) for k in ("gravity", "magnetic")]
EDGE = [
    (1, 1, 1, [0, 0, 0, 0]),      # a single station over a single prism
    (1, 37, 2, [2, 3, 0, 1]),     # one station column
    (45, 1, 2, [0, 1, 4, 4]),     # one station row
    (64, 3, 3, [0, 0, 0, 0]),     # power-of-two embedding in x
]


def check(sx, sy, nz, pads, dx, dy, z, kind, dtype, seed):
    og = O.ogrid(sx, sy, nz, *pads, dx, dy, list(z))
    if kind == "gravity":
        params, oargs = B.KernelParams.gravity(), ("gravity", O.grav_constants())
    else:
        params = B.KernelParams.magnetic(17.0, 55.0, 48000.0)
        oargs = ("magnetic", O.mag_constants(17.0, 55.0, 48000.0))
    fw, tr = O.build_spectra(og, *oargs)
    rng = np.random.default_rng(100 + seed)
    x = np.asarray(rng.uniform(0.0, 1.0, og.n), dtype=dtype).astype(np.float64)
    v = np.asarray(rng.normal(0.0, 1.0, og.m), dtype=dtype).astype(np.float64)
    grid = B.make_grid(sx, sy, nz, *pads, dx, dy, z)
    with B.build_transform_stack(grid, params, dtype=dtype) as st:
        f = B.apply(st, x, "forward")
        t = B.apply(st, v, "transpose")
    ef = O.rel_l2(O.forward(og, fw, x), f)
    et = O.rel_l2(O.transpose(og, tr, v), t)
    assert ef <= TOL[dtype], (sx, sy, nz, pads, st.fft_shape, ef)
    assert et <= TOL[dtype], (sx, sy, nz, pads, st.fft_shape, et)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("seed,kind", CASES)
def test_random_geometries(seed, kind, dtype):
    sx, sy, nz, pads, dx, dy, z = draw(seed)
    check(sx, sy, nz, pads, dx, dy, z, kind, dtype, seed)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("case", EDGE, ids=["1x1x1", "sx1", "sy1", "pow2x"])
def test_edge_geometries(case, dtype):
    sx, sy, nz, pads = case
    z = np.linspace(0.0, 40.0 * nz, nz + 1)
    for kind in ("gravity", "magnetic"):
        check(sx, sy, nz, pads, 25.0, 30.0, z, kind, dtype, sx * 31 + sy)
