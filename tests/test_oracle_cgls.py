"""CPU pin of the oracle's CGLS (the checker of bttb_cgls).

CGLS from m = 0 stays in range(G^T), so it converges to the minimum-norm
least-squares solution pinv(G) d; on a grid small enough for the dense
per-entry operator it must reach it.  With damping it converges to the
Tikhonov solution (G^T G + damp^2 I)^-1 G^T d.
"""
import numpy as np
import pytest

from oracle import bttb_oracle as O


@pytest.mark.parametrize("damp", [0.0, 0.3])
def test_oracle_cgls_converges_to_least_squares(damp):
    og = O.ogrid(4, 3, 2, 1, 1, 0, 1, 1.0, 1.5, (0.0, 1.0, 2.5))
    gs = O.grav_constants(scale=3e9)  # singular values of order 1: a well-scaled toy system
    fw, tr = O.build_spectra(og, "gravity", gs)
    G = np.hstack(O.dense_layers(og, "gravity", gs))
    d = np.random.default_rng(0).normal(size=og.m)
    m, hist = O.cgls(og, fw, tr, d, 60, damp)
    if damp == 0.0:
        want = np.linalg.pinv(G) @ d
    else:
        want = np.linalg.solve(G.T @ G + damp * damp * np.eye(og.n), G.T @ d)
    assert O.rel_l2(want, m) <= 1e-8
    assert len(hist) == 61 and hist[0] == pytest.approx(np.linalg.norm(d))
    np.testing.assert_allclose(hist[-1], np.linalg.norm(d - G @ m), rtol=1e-8, atol=1e-12)
