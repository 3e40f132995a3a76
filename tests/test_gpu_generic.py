"""Generic-length path (csrc/generic.cu): embeddings above the shared-memory
engine's 8192 (the reference has no size cap: grid.py:101-104 embed_shape,
transform.py:101 np.fft.fft2 of any shape; VERDICT r1 missing 3).

* BTTB_GENERIC=1 forces every plan onto the generic path, so it is pinned on
  the same small cases as the main path: the reference's own padded 6x5x2
  products (tests/golden) and the C1-C3 configs against the oracle.
* Real > 8192 embeddings: 4300 x 3 and 4200 x 40 station lines (embedding
  8599 -> FFT length 8640 = 2^6 3^3 5) against the oracle.
"""
import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-10, "float32": 1e-5}
GRAV = B.KernelParams.gravity()
MAG = B.KernelParams.magnetic(33.0, 47.0, 45000.0)


def bgrid(og):
    return B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)


def oparams(params):
    return (params.kind, params.gamma * params.scale if params.kind == "gravity" else np.array(params.gc))


def q(a, dtype):
    return np.asarray(a, dtype=dtype).astype(np.float64)


@pytest.fixture
def forced(monkeypatch):
    monkeypatch.setenv("BTTB_GENERIC", "1")


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("pads", [(0, 0, 0, 0), (2, 1, 1, 2), (3, 0, 0, 2)])
@pytest.mark.parametrize("params", [GRAV, MAG], ids=["gravity", "magnetic"])
def test_forced_generic_small_grids_vs_reference(forced, golden, dtype, pads, params):
    z = golden("small_6x5x2.npz")
    key = f"{params.kind}_{'_'.join(map(str, pads))}"
    g = B.make_grid(6, 5, 2, *pads, 1.0, 1.5, (0.0, 1.0, 2.5))
    u, v = z[f"{key}/u"], z[f"{key}/v"]
    with B.build_transform_stack(g, params, dtype=dtype) as st:
        f = B.apply(st, u, "forward")
        t = B.apply(st, v, "transpose")
    og = O.ogrid(6, 5, 2, *pads, 1.0, 1.5, (0.0, 1.0, 2.5))
    fw, tr = O.build_spectra(og, *oparams(params))
    assert O.rel_l2(O.forward(og, fw, q(u, dtype)), f) <= TOL[dtype]
    assert O.rel_l2(O.transpose(og, tr, q(v, dtype)), t) <= TOL[dtype]
    if dtype == "float64":
        assert B.relative_error(z[f"{key}/fwd"], f) <= 1e-10
        assert B.relative_error(z[f"{key}/tra"], t) <= 1e-10


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_forced_generic_configs_vs_oracle(forced, monkeypatch, cfg, dtype):
    og = O.config_grid(cfg)
    kind, consts = O.config_kernel(cfg)
    params = GRAV if kind == "gravity" else B.KernelParams.magnetic(*O.CONFIGS[cfg][11])
    x, d = O.make_inputs(cfg, og, batch=2)
    fw, tr = O.build_spectra(og, kind, consts)
    with B.build_transform_stack(bgrid(og), params, dtype=dtype) as st:
        f = B.apply(st, x, "forward")
        t = B.apply(st, d, "transpose")
        lx, ly = st.fft_shape
        spec = st.layer_spectrum(0)
    for b in range(2):
        assert O.rel_l2(O.forward(og, fw, q(x[b], dtype)), f[b]) <= TOL[dtype]
        assert O.rel_l2(O.transpose(og, tr, q(d[b], dtype)), t[b]) <= TOL[dtype]
    # the same cached half spectrum as a main-path plan at the same lengths
    monkeypatch.delenv("BTTB_GENERIC")
    with B.build_transform_stack(bgrid(og), params, dtype=dtype, fft_shape=(lx, ly)) as st2:
        ref = st2.layer_spectrum(0)
    tol = (1e-12 if dtype == "float64" else 1e-6) * np.abs(ref).max()
    np.testing.assert_allclose(spec, ref, rtol=0, atol=tol)


def test_forced_generic_cgls_and_staged(forced):
    og = O.config_grid("C1")
    fw, tr = O.build_spectra(og, *O.config_kernel("C1"))
    d = np.random.default_rng(2).normal(size=og.m)
    with B.build_transform_stack(bgrid(og), GRAV) as st:
        m, hist = B.cgls(st, d, iters=4)
        from paper_1912_06976_b200.parallel import DeviceOperator
        import torch
        with pytest.raises(Exception, match="split products"):
            DeviceOperator(st).forward_spectrum(torch.zeros(og.n, dtype=torch.float64, device="cuda"))
    m_ref, h_ref = O.cgls(og, fw, tr, d, 4)
    assert O.rel_l2(m_ref, m) <= 1e-10
    np.testing.assert_allclose(hist, h_ref, rtol=1e-10)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("sy,params", [(3, MAG), (40, GRAV)], ids=["4300x3-magnetic", "4200x40-gravity"])
def test_embedding_above_8192(dtype, sy, params):
    sx = 4300 if sy == 3 else 4200
    og = O.ogrid(sx, sy, 2, 0, 0, 0, 0, 10.0, 10.0, [0.0, 10.0, 25.0])
    assert og.mx > 8192
    rng = np.random.default_rng(8)
    x = rng.uniform(0.0, 1.0, og.n)
    v = rng.normal(0.0, 1.0, og.m)
    with B.build_transform_stack(bgrid(og), params, dtype=dtype) as st:
        assert st.fft_shape[0] == B.fft_length(og.mx) == 8640
        f = B.apply(st, x, "forward")
        t = B.apply(st, v, "transpose")
    fw, tr = O.build_spectra(og, *oparams(params))
    assert O.rel_l2(O.forward(og, fw, q(x, dtype)), f) <= TOL[dtype]
    assert O.rel_l2(O.transpose(og, tr, q(v, dtype)), t) <= TOL[dtype]
