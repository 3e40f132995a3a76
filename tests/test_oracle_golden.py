"""Pin the CPU oracle (oracle/bttb_oracle.py) to the reference implementation.

The golden vectors in tests/golden/ were produced by the reference package
itself (tests/golden/make_golden.py imports /root/reference/pkg/src/bttb);
the oracle must reproduce them BIT-FOR-BIT, which is what licenses it as the
parity checker for the GPU path on machines without the reference.
Known-answer values are the reference tests' own (pkg/tests/oracles.py:104,
pkg/tests/test_kernels.py:23-38, :84-91, :101-114).
"""
import math

import numpy as np
import pytest

from oracle import bttb_oracle as O

PADS = [(0, 0, 0, 0), (1, 1, 1, 1), (2, 1, 1, 2), (3, 0, 0, 2)]
KERNELS = [("gravity", O.grav_constants()), ("magnetic", O.mag_constants(33.0, 47.0, 45000.0))]


@pytest.mark.parametrize("pads", PADS)
@pytest.mark.parametrize("kind,consts", KERNELS, ids=["gravity", "magnetic"])
def test_small_grids_bit_identical(golden, pads, kind, consts):
    z = golden("small_6x5x2.npz")
    g = O.ogrid(6, 5, 2, *pads, 1.0, 1.5, (0.0, 1.0, 2.5))
    key = f"{kind}_{'_'.join(map(str, pads))}"
    for r in range(g.nz):
        assert np.array_equal(O.layer_window(g, kind, consts, r), z[f"{key}/window{r}"])
    fw, tr = O.build_spectra(g, kind, consts)
    assert np.array_equal(O.forward(g, fw, z[f"{key}/u"]), z[f"{key}/fwd"])
    assert np.array_equal(O.transpose(g, tr, z[f"{key}/v"]), z[f"{key}/tra"])


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_baseline_configs_bit_identical(golden, name):
    G = golden(f"{name}.npz")
    g = O.config_grid(name)
    kind, consts = O.config_kernel(name)
    x, d = O.make_inputs(name, g, batch=1)
    assert np.linalg.norm(x) == G["x_norm"] and np.linalg.norm(d) == G["d_norm"]
    assert np.array_equal(O.layer_window(g, kind, consts, 0), G["window_top"])
    assert np.array_equal(O.layer_window(g, kind, consts, g.nz - 1), G["window_bottom"])
    fw, tr = O.build_spectra(g, kind, consts)
    assert np.array_equal(O.forward(g, fw, x[0]), G["fwd"])
    t = O.transpose(g, tr, d[0])
    assert np.array_equal(t[::int(G["tra_sub"])], G["tra"])
    assert np.linalg.norm(t) == G["tra_norm"]


def test_c4_windows_sampled_bit_identical(golden):
    G = golden("C4_windows.npz")
    g = O.config_grid("C4")
    kind, consts = O.config_kernel("C4")
    for r in (0, g.nz - 1):
        w = O.layer_window(g, kind, consts, r)
        assert np.array_equal(w[G["ia"], G["ib"]], G[f"w{r}"])
        assert np.linalg.norm(w) == G[f"w{r}_norm"]


def _unit_quadrature(n):
    # midpoint rule of gamma*z/r^3 over the unit cube z in [1/2, 3/2] (independent check)
    h = 1.0 / n
    xs = -0.5 + (np.arange(n) + 0.5) * h
    tot = 0.0
    for z in 0.5 + (np.arange(n) + 0.5) * h:
        r2 = xs[:, None] ** 2 + xs[None, :] ** 2 + z * z
        tot += np.sum(z / r2 ** 1.5)
    return O.GAMMA * tot * h ** 3


UNIT_CUBE_FROZEN = 6.293849964187017e-11  # pkg/tests/oracles.py:104


def test_known_answer_unit_cube():
    assert abs(_unit_quadrature(64) - UNIT_CUBE_FROZEN) / UNIT_CUBE_FROZEN < 1e-6
    val = O.gravity_corner_sum(0.5, 1.5, np.array([-0.5, 0.5]), np.array([-0.5, 0.5]), O.GAMMA)[0, 0]
    assert abs(val - UNIT_CUBE_FROZEN) / UNIT_CUBE_FROZEN < 5e-7


def test_known_answer_bouguer_slab():
    c = np.arange(-50.5, 51.0, 1.0)
    s = O.gravity_corner_sum(0.1, 0.2, c, c, O.GAMMA).sum()
    ref = 2.0 * math.pi * O.GAMMA * 0.1
    assert abs(s - ref) / ref < 0.01


@pytest.mark.parametrize("D,I", [(33.0, 47.0), (0.0, 90.0), (120.0, -35.0)])
def test_known_answer_far_field_dipole(D, I):
    gc = O.mag_constants(D, I, 45000.0)
    xa, xb, ya, yb, z1, z2 = 40.25, 41.25, -25.75, -24.75, 10.0, 11.0
    got = O.magnetic_entries(z1, z2, np.array([xa, xb]), np.array([ya, yb]), gc)[0, 0]
    f = np.array([math.cos(math.radians(I)) * math.cos(math.radians(D)),
                  math.cos(math.radians(I)) * math.sin(math.radians(D)), math.sin(math.radians(I))])
    r = np.array([-(xa + xb) / 2, -(ya + yb) / 2, -(z1 + z2) / 2])
    rn = np.linalg.norm(r)
    ref = (45000.0 / (4 * math.pi)) * (3 * np.dot(f, r / rn) ** 2 - 1) / rn ** 3
    assert abs(got - ref) / abs(ref) < 0.01


def test_known_answer_direction_cosines():
    ht = 50000.0 / (4 * math.pi)
    np.testing.assert_allclose(O.mag_constants(0.0, 90.0, 50000.0), [0, 0, 0, ht, ht], atol=1e-9)
    np.testing.assert_allclose(O.mag_constants(0.0, 0.0, 50000.0), [0, 0, 0, 0, -ht], atol=1e-9)


def test_zero_thickness_exact_zero():
    c = np.array([-0.5, 0.5, 1.5, 2.5])
    assert np.all(O.gravity_corner_sum(1.0, 1.0, c, c[:3], O.GAMMA) == 0.0)
    assert np.all(O.magnetic_entries(1.0, 1.0, c, c[:3], O.mag_constants(33, 47, 45000.0)) == 0.0)


def test_rel_l2_semantics():
    assert O.rel_l2([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert O.rel_l2([3.0, 4.0], [0.0, 0.0]) == 1.0
    assert O.rel_l2([0.0, 0.0], [0.0, 0.0]) == 0.0
    assert O.rel_l2([0.0, 0.0], [0.0, 1.0]) == np.inf
    with pytest.raises(ValueError, match="shape"):
        O.rel_l2(np.zeros(2), np.zeros(3))
