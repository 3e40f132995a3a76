"""Host-side mirror of the reference API: validation, geometry, messages.

Mirrors the reference's own unit tests of these contracts
(pkg/tests/test_grid.py, test_kernels.py:117-128, test_multiply.py:95-113,
test_transform.py:26-80, test_acceptance.py:58-77) on the drop-in package.
"""
import numpy as np
import pytest

import paper_1912_06976_b200 as B
from paper_1912_06976_b200 import multiply
from paper_1912_06976_b200.parallel import partition_layers


def test_grid_derived_sizes():
    g = B.make_grid(25, 15, 2, 1, 1, 1, 1, 100.0, 100.0, (0, 100, 200))
    assert (g.nx, g.ny, g.m, g.n_r, g.n) == (27, 17, 375, 459, 918)
    assert g.embed_shape == (51, 31)
    g = B.make_grid(1, 1, 1, 0, 0, 0, 0, 1.0, 1.0, (0.0, 1.0))
    assert (g.m, g.n) == (1, 1)


@pytest.mark.parametrize("args,field", [
    ((0, 3, 1, 0, 0, 0, 0, 1.0, 1.0, (0, 1)), "sx"),
    ((2, 0, 1, 0, 0, 0, 0, 1.0, 1.0, (0, 1)), "sy"),
    ((2, 3, 0, 0, 0, 0, 0, 1.0, 1.0, (0,)), "nz"),
    ((2, 3, 1, -1, 0, 0, 0, 1.0, 1.0, (0, 1)), "pxl"),
    ((2, 3, 1, 0, 0, 0, 0, 0.0, 1.0, (0, 1)), "dx"),
    ((2, 3, 1, 0, 0, 0, 0, 1.0, -1.0, (0, 1)), "dy"),
    ((2, 3, 2, 0, 0, 0, 0, 1.0, 1.0, (0, 1)), "z_blocks"),
    ((2, 3, 2, 0, 0, 0, 0, 1.0, 1.0, (0, 2, 1)), "z_blocks"),
    ((2, 3, 1, 0, 0, 0, 0, 1.0, 1.0, (-1, 1)), "z_blocks"),
])
def test_grid_validation_names_the_field(args, field):
    with pytest.raises(ValueError, match=field):
        B.make_grid(*args)


def test_scaled_problem_table():
    # Table 1 of the paper (reference pkg/tests/test_acceptance.py:58-77)
    m_ref = (375, 1500, 3375, 6000, 9375, 13500, 18375, 24000, 30375, 37500, 45375, 54000)
    n0 = (750, 6000, 20250, 48000, 93750, 162000, 257250, 384000, 546750, 750000, 998250, 1296000)
    n5 = (918, 7616, 24402, 58080, 113710, 199200, 310730, 464640, 662454, 916320, 1206546, 1568160)
    for k in range(12):
        assert B.scaled_problem(k + 1, 0.0).m == m_ref[k]
        assert B.scaled_problem(k + 1, 0.0).n == n0[k]
        assert B.scaled_problem(k + 1, 0.05).n == n5[k]


def test_distance_tables():
    g = B.make_grid(2, 2, 1, 0, 0, 0, 0, 1.0, 1.0, (0, 1))
    np.testing.assert_array_equal(B.sym_distances(g).x, [-0.5, 0.5, 1.5])
    np.testing.assert_array_equal(B.full_distances(g).x, [-1.5, -0.5, 0.5, 1.5])
    g = B.make_grid(4, 2, 1, 2, 1, 0, 0, 1.0, 1.0, (0, 1))
    assert B.sym_distances(g).x.size == 7 and B.full_distances(g).x.size == 12
    t = B.sym_distances(g)
    np.testing.assert_array_equal(t.r2, t.x[:, None] ** 2 + t.y[None, :] ** 2)
    assert not t.x.flags.writeable


def test_kernel_params_and_constants():
    ht = 50000.0 / (4 * np.pi)
    np.testing.assert_allclose(B.magnetic_constants(0.0, 90.0, 50000.0), [0, 0, 0, ht, ht], atol=1e-9)
    with pytest.raises(ValueError, match="F"):
        B.magnetic_constants(0.0, 45.0, 0.0)
    with pytest.raises(ValueError, match="gamma"):
        B.KernelParams.gravity(gamma=0.0)
    k = B.KernelParams.magnetic(33.0, 47.0, 45000.0).native()
    assert k.kind == 1 and list(k.gc) == list(B.magnetic_constants(33.0, 47.0, 45000.0))
    k = B.KernelParams.gravity(scale=1e5).native()
    assert k.kind == 0 and k.gamma_scaled == B.GRAVITATIONAL_CONST * 1e5


class _FakeStack:
    """Duck-typed stack for host-side validation (no device plan needed)."""

    def __init__(self, g):
        self.grid = g
        self.nz_local = g.nz
        self.n_local = g.n
        self.dtype = np.dtype(np.float64)
        self.handle = None


def test_apply_validation_messages():
    g = B.make_grid(6, 5, 2, 1, 1, 1, 1, 1.0, 1.5, (0.0, 1.0, 2.5))
    st = _FakeStack(g)
    with pytest.raises(ValueError, match=rf"n={g.n}"):
        multiply.apply(st, np.zeros(g.n - 1), "forward")
    with pytest.raises(ValueError, match=r"nx\*ny\*nz = 8\*7\*2"):
        multiply.apply(st, np.zeros(g.n - 1), "forward")
    with pytest.raises(ValueError, match=rf"m={g.m}"):
        multiply.apply(st, np.zeros(g.m + 2), "transpose")
    with pytest.raises(ValueError, match="mode"):
        multiply.apply(st, np.zeros(g.n), "backward")


def test_simulate_validation_message():
    g = B.make_grid(3, 2, 2, 0, 0, 0, 0, 1.0, 1.0, (0, 1, 2))
    with pytest.raises(ValueError, match=r"n=12 = nx\*ny\*nz = 3\*2\*2"):
        B.simulate(g, B.KernelParams.gravity(), np.zeros(5))


def test_relative_error_known_answers():
    assert B.relative_error(np.array([1.0, 2.0]), np.array([1.0, 2.0])) == 0.0
    assert B.relative_error(np.array([3.0, 4.0]), np.array([0.0, 0.0])) == 1.0
    assert B.relative_error(np.array([1.0, 0.0]), np.array([1.0, 1e-13])) == pytest.approx(1e-13)
    assert B.relative_error(np.zeros(2), np.array([0.0, 1.0])) == np.inf
    with pytest.raises(ValueError, match="shape"):
        B.relative_error(np.zeros(2), np.zeros(3))


def test_transpose_layout_and_extension_column():
    T = np.array([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0], [7.0, 8.0, 9.0]])
    np.testing.assert_array_equal(B.transpose_layout(T), [[1, 3, 2], [7, 9, 8], [4, 6, 5]])
    R = np.random.default_rng(1).uniform(size=(6, 9))
    np.testing.assert_array_equal(B.transpose_layout(B.transpose_layout(R)), R)
    np.testing.assert_array_equal(B.circulant_extension_column([1.0, 10.0, 11.0], [1.0, 2.0, 3.0]),
                                  [1.0, 10.0, 11.0, 3.0, 2.0])
    with pytest.raises(ValueError, match="corner"):
        B.circulant_extension_column(np.array([1.0, 2.0]), np.array([3.0, 4.0]))


def test_partition_layers():
    assert partition_layers(20, 8) == [(0, 3), (3, 6), (6, 9), (9, 12), (12, 14), (14, 16), (16, 18), (18, 20)]
    assert partition_layers(128, 8)[-1] == (112, 128)
    assert partition_layers(5, 1) == [(0, 5)]
    with pytest.raises(ValueError):
        partition_layers(3, 4)


def test_product_package_does_not_import_the_oracle():
    import subprocess
    import sys
    code = ("import sys, paper_1912_06976_b200 as B; "
            "import paper_1912_06976_b200.parallel, paper_1912_06976_b200.harness; "
            "assert not any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules), "
            "[m for m in sys.modules if m.startswith('oracle')]")
    subprocess.run([sys.executable, "-c", code], check=True,
                   cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))


def test_bench_csv_schema_matches_reference_columns():
    # harness.py:20-43 of the reference: same columns, same float format, "" for None
    from paper_1912_06976_b200.harness import CSV_COLUMNS, BenchRecord, bench_csv_text

    assert CSV_COLUMNS == ("schema_version", "problem", "padding", "kernel", "path", "phase",
                           "trials", "mean_seconds", "mean_rel_error_vs_dense", "m", "n", "seed")
    rec = BenchRecord(problem=2, padding=0.1, kernel="gravity", path="transform", phase="forward",
                      trials=5, mean_seconds=1.5e-3, mean_rel_error=None, m=1500, n=8640, seed=0)
    lines = bench_csv_text([rec]).splitlines()
    assert lines[0] == ",".join(CSV_COLUMNS)
    assert lines[1] == "1,2,0.1,gravity,transform,forward,5,1.500000000e-03,,1500,8640,0"


def test_cli_bench_rejects_bad_problem_index(capsys):
    from paper_1912_06976_b200 import cli

    assert cli.main(["bench", "--problems", "13"]) == 2
    assert "unknown problem index 13" in capsys.readouterr().err


def test_bench_profile_figures_are_tied_to_the_kernel_sources(tmp_path, monkeypatch):
    """bench.py reports a committed ncu figure (DRAM traffic, FP64-pipe floor)
    only while the CUDA sources hash to the digest the profile was taken on."""
    import json

    import bench

    prof = tmp_path / "profiles"
    prof.mkdir()
    cur = bench.csrc_digest()
    (prof / "traffic.json").write_text(json.dumps({
        "C4_f64": {"bytes_per_apply": 9.5e9, "profile": "rX", "csrc_sha": cur},
        "C4_f32": {"bytes_per_apply": 4.7e9, "profile": "rOld", "csrc_sha": "0" * 16}}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "csrc_digest", lambda: cur)
    val, src = bench.measured_traffic("C4", "f64")
    assert val == 9.5e9 and src["profile"] == "rX" and not src.get("stale")
    val, src = bench.measured_traffic("C4", "f32")
    assert val is None and src["stale"] is True
    assert bench.profile_record("missing") == (None, None)
