"""Size-independent properties at BASELINE sizes, where the oracle is too slow.

Full C4 (1000x1000x128, 2048x2048 FFTs of the 1999x1999 embedding): adjoint identity, linearity, zero ->
zero, layer-shard additivity.  Adjoint bound as in pkg/tests/test_multiply.py:54-66.
"""
import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

GRAV = B.KernelParams.gravity()
MAG = B.KernelParams.magnetic(33.0, 47.0, 45000.0)


def c4():
    og = O.config_grid("C4")
    g = B.make_grid(og.sx, og.sy, og.nz, 0, 0, 0, 0, og.dx, og.dy, og.z)
    return g, B.KernelParams.magnetic(*O.CONFIGS["C4"][11])


@pytest.fixture(scope="module")
def c4_stack():
    g, p = c4()
    st = B.build_transform_stack(g, p)
    yield g, st
    st.close()


def test_c4_adjoint_identity(c4_stack):
    g, st = c4_stack
    rng = np.random.default_rng(21)
    u = rng.uniform(0.0, 0.05, g.n)
    v = rng.normal(0.0, 1.0, g.m)
    lhs = np.dot(B.apply(st, u, "forward"), v)
    rhs = np.dot(u, B.apply(st, v, "transpose"))
    assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(u) * np.linalg.norm(v) * np.sqrt(g.m * g.n)
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs))


def test_c4_linearity_and_zero(c4_stack):
    g, st = c4_stack
    rng = np.random.default_rng(22)
    u, w = rng.uniform(size=(2, g.n))
    a, b = 2.25, -0.75
    comb = B.apply(st, a * u + b * w, "forward")
    split = a * B.apply(st, u, "forward") + b * B.apply(st, w, "forward")
    assert B.relative_error(comb, split) <= 1e-12
    assert np.all(B.apply(st, np.zeros(g.n), "forward") == 0.0)
    assert np.all(B.apply(st, np.zeros(g.m), "transpose") == 0.0)


def test_c4_layer_shards_add_up(c4_stack):
    g, st = c4_stack
    _, p = c4()
    rng = np.random.default_rng(23)
    u = rng.uniform(0.0, 0.05, g.n)
    v = rng.normal(0.0, 1.0, g.m)
    full_f = B.apply(st, u, "forward")
    full_t = B.apply(st, v, "transpose")
    parts_f, parts_t = [], []
    for lo, hi in ((0, 50), (50, 128)):
        with B.build_transform_stack(g, p, layers=(lo, hi)) as sh:
            parts_f.append(B.apply(sh, u[lo * g.n_r:hi * g.n_r], "forward"))
            parts_t.append(B.apply(sh, v, "transpose"))
    assert B.relative_error(full_f, parts_f[0] + parts_f[1]) <= 1e-13
    np.testing.assert_array_equal(np.concatenate(parts_t), full_t)


@pytest.mark.parametrize("params", [GRAV, MAG], ids=["gravity", "magnetic"])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_adjoint_identity_scaled_problems(params, k):
    g = B.scaled_problem(k, 0.05 if k != 2 else 0.0)
    rng = np.random.default_rng(6)
    with B.build_transform_stack(g, params) as st:
        for _ in range(3):
            u = rng.uniform(size=g.n)
            v = rng.uniform(size=g.m)
            gap = abs(np.dot(B.apply(st, u, "forward"), v) - np.dot(u, B.apply(st, v, "transpose")))
            assert gap <= 1e-10 * np.linalg.norm(u) * np.linalg.norm(v) * np.sqrt(g.m * g.n)


def test_dimension_mismatch_errors():
    g = B.make_grid(6, 5, 2, 1, 1, 1, 1, 1.0, 1.5, (0.0, 1.0, 2.5))
    with B.build_transform_stack(g, GRAV) as st:
        with pytest.raises(ValueError, match=rf"n={g.n}"):
            B.apply(st, np.zeros(g.n - 1), "forward")
        with pytest.raises(ValueError, match=rf"m={g.m}"):
            B.apply(st, np.zeros(g.m + 2), "transpose")
        with pytest.raises(ValueError, match="mode"):
            B.apply(st, np.zeros(g.n), "backward")


def test_torch_device_path_matches_host_path():
    import torch
    og = O.config_grid("C3")
    g = B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)
    x, d = O.make_inputs("C3", og, batch=2)
    for dtype in ("float64", "float32"):
        with B.build_transform_stack(g, GRAV, dtype=dtype) as st:
            fh = B.apply(st, x, "forward")
            th = B.apply(st, d, "transpose")
            tdt = torch.float64 if dtype == "float64" else torch.float32
            fd = B.apply(st, torch.tensor(x, dtype=tdt, device="cuda"), "forward")
            td = B.apply(st, torch.tensor(d, dtype=tdt, device="cuda"), "transpose")
            np.testing.assert_array_equal(fd.cpu().numpy(), fh)
            np.testing.assert_array_equal(td.cpu().numpy(), th)


def test_spectrum_is_hermitian_consistent_and_cached():
    og = O.config_grid("C2")
    g = B.make_grid(og.sx, og.sy, og.nz, 0, 0, 0, 0, og.dx, og.dy, og.z)
    p = B.KernelParams.magnetic(*O.CONFIGS["C2"][11])
    with B.build_transform_stack(g, p) as st:
        S = st.layer_spectrum(0)
        Lx, Ly = st.fft_shape
        assert S.shape == (Lx // 2 + 1, Ly)
        # the kx = 0 column of the half spectrum of a real array is Hermitian in ky
        col = S[0]
        np.testing.assert_allclose(col[1:], np.conj(col[1:][::-1]), rtol=0, atol=1e-12 * np.abs(col).max())
        assert st.element_count == g.nz * g.embed_shape[0] * g.embed_shape[1]
        assert st.device_bytes == g.nz * (Lx // 2 + 1) * Ly * 16


def test_cli_bench_writes_transform_gpu_rows(tmp_path):
    import csv

    from paper_1912_06976_b200 import cli

    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--problems", "1-2", "--trials", "2", "--padding", "0.1", "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert [(r["problem"], r["phase"]) for r in rows] == [
        ("1", "build"), ("1", "forward"), ("1", "transpose"), ("2", "build"), ("2", "forward"), ("2", "transpose")]
    assert all(r["path"] == "transform-gpu" and r["mean_rel_error_vs_dense"] == "" for r in rows)
    assert all(float(r["mean_seconds"]) > 0 for r in rows)
