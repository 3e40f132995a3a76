"""Device-resident batched CGLS (bttb_cgls) against the
oracle's CGLS over the pinned CPU operator.

Gates: the iterates of a Krylov method amplify the operator's last-bit
differences with the iteration count, so the CGLS gates are looser than the
single-product gates of test_gpu_parity.py: models and residual histories
within relative 1e-8 (fp64) / 2e-3 (fp32) of the oracle after 8 iterations.
"""
import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-8, "float32": 2e-3}


def bgrid(og):
    return B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("damp", [0.0, 3e-6])
@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_cgls_matches_oracle(kind, damp, dtype):
    og = O.ogrid(24, 20, 4, 2, 1, 1, 2, 50.0, 40.0, [0.0, 30.0, 60.0, 100.0, 150.0])
    if kind == "gravity":
        params, oparams = B.KernelParams.gravity(), ("gravity", O.grav_constants())
    else:
        params = B.KernelParams.magnetic(10.0, 60.0, 50000.0)
        oparams = ("magnetic", O.mag_constants(10.0, 60.0, 50000.0))
    fw, tr = O.build_spectra(og, *oparams)
    rng = np.random.default_rng(5)
    truth = rng.uniform(0, 1, (3, og.n))
    d = np.stack([O.forward(og, fw, t) for t in truth])
    d = np.asarray(d, dtype=dtype).astype(np.float64)
    # damping scaled to the operator (gravity entries ~1e-6, magnetic ~1e2)
    dmp = damp * (1.0 if kind == "gravity" else 1e8)
    with B.build_transform_stack(bgrid(og), params, dtype=dtype) as st:
        m, hist = B.cgls(st, d, iters=8, damp=dmp)
    assert m.shape == (3, og.n) and hist.shape == (3, 9)
    for b in range(3):
        mo, ho = O.cgls(og, fw, tr, d[b], 8, dmp, rtol=1e-13 if dtype == "float64" else 1e-6)
        assert O.rel_l2(mo, m[b]) <= TOL[dtype]
        np.testing.assert_allclose(hist[b], ho, rtol=TOL[dtype])
        if dmp == 0.0:
            assert np.all(np.diff(hist[b]) <= 1e-12 * hist[b][0])  # CGLS residuals never grow


def test_cgls_zero_iterations_and_single_vector():
    og = O.ogrid(10, 8, 2, 0, 0, 0, 0, 50.0, 50.0, [0.0, 50.0, 100.0])
    d = np.random.default_rng(1).normal(size=og.m)
    with B.build_transform_stack(bgrid(og), B.KernelParams.gravity()) as st:
        m0, h0 = B.cgls(st, d, iters=0)
        assert m0.shape == (og.n,) and np.all(m0 == 0.0)
        np.testing.assert_allclose(h0, [np.linalg.norm(d)], rtol=1e-14)
        m1, h1 = B.cgls(st, np.zeros(og.m), iters=3)
        assert np.all(m1 == 0.0) and np.all(h1 == 0.0)


def test_cgls_batch_items_independent():
    og = O.ogrid(16, 12, 3, 0, 0, 0, 0, 50.0, 50.0, [0.0, 50.0, 100.0, 150.0])
    d = np.random.default_rng(2).normal(size=(4, og.m))
    with B.build_transform_stack(bgrid(og), B.KernelParams.gravity()) as st:
        mb, hb = B.cgls(st, d, iters=5)
        for b in range(4):
            ms, hs = B.cgls(st, d[b], iters=5)
            assert O.rel_l2(ms, mb[b]) <= 1e-12
            np.testing.assert_allclose(hs, hb[b], rtol=1e-12)


def test_cgls_torch_device_path():
    torch = pytest.importorskip("torch")
    og = O.ogrid(16, 12, 3, 1, 1, 1, 1, 50.0, 50.0, [0.0, 50.0, 100.0, 150.0])
    d = np.random.default_rng(3).normal(size=(2, og.m))
    with B.build_transform_stack(bgrid(og), B.KernelParams.gravity(), dtype="float32") as st:
        mh, hh = B.cgls(st, d, iters=4)
        md, hd = B.cgls(st, torch.tensor(d, device="cuda:0"), iters=4)
        torch.cuda.synchronize()
    assert md.is_cuda and md.dtype == torch.float32
    np.testing.assert_array_equal(md.cpu().numpy(), mh)
    np.testing.assert_array_equal(hd, hh)


def test_cgls_rejects_bad_arguments_and_layer_shards():
    og = O.ogrid(10, 8, 2, 0, 0, 0, 0, 50.0, 50.0, [0.0, 50.0, 100.0])
    with B.build_transform_stack(bgrid(og), B.KernelParams.gravity()) as st:
        with pytest.raises(ValueError, match="m=80"):
            B.cgls(st, np.zeros(79))
        with pytest.raises(ValueError, match="iters"):
            B.cgls(st, np.zeros(og.m), iters=-1)
        with pytest.raises(ValueError, match="damp"):
            B.cgls(st, np.zeros(og.m), damp=-1.0)
    with B.build_transform_stack(bgrid(og), B.KernelParams.gravity(), layers=(1, 2)) as st:
        with pytest.raises(ValueError, match="every layer"):
            B.cgls(st, np.zeros(og.m))
