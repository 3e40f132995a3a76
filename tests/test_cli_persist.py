"""CLI, vector files and stack persistence.

Mirrors the reference's tests of these contracts (pkg/tests/test_cli.py:105-217,
pkg/tests/test_transform.py:144-176, test_acceptance.py:185-198) on the
drop-in; CPU tests need no GPU, the rest are marked gpu.
"""
import os

import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O
from paper_1912_06976_b200.cli import main

GRID_FLAGS = ["--sx", "4", "--sy", "3", "--nz", "2", "--pxl", "1", "--pxr", "0",
              "--pyl", "0", "--pyr", "1", "--dx", "1.0", "--dy", "1.5", "--zblocks", "0,1,2.5"]
GRID = B.make_grid(4, 3, 2, 1, 0, 0, 1, 1.0, 1.5, (0.0, 1.0, 2.5))


@pytest.mark.parametrize("ext", ["txt", "bin"])
def test_vector_round_trip(tmp_path, ext):
    path = str(tmp_path / f"v.{ext}")
    x = np.random.default_rng(9).uniform(size=33)
    B.write_vector(x, path)
    np.testing.assert_array_equal(B.read_vector(path), x)


def test_vector_unknown_extension(tmp_path):
    with pytest.raises(ValueError, match="txt"):
        B.write_vector(np.zeros(3), str(tmp_path / "v.dat"))


def test_sizes_command(tmp_path):
    out = tmp_path / "sizes.csv"
    assert main(["sizes", "--padding", "0.05", "--out", str(out)]) == 0
    rows = out.read_text().strip().splitlines()
    assert rows[0].startswith("problem,") and len(rows) == 13
    hdr = rows[0].split(",")
    first = dict(zip(hdr, rows[1].split(",")))
    # the reference's columns (harness.py:55-64), then the GPU plan's FFT shape and cache bytes
    assert hdr[:10] == ["problem", "sx", "sy", "nz", "pxl", "pyl", "nx", "ny", "m", "n"]
    assert first["n"] == "918" and first["gpu_fft_shape"] == "64x32"


def test_unknown_config_key_rejected(tmp_path, capsys):
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("sx = 4\nbogus = 1\n")
    assert main(["simulate", "--config", str(cfg), "--model", "x.txt", "--out", "y.txt"]) == 2
    assert "bogus" in capsys.readouterr().err


def test_missing_grid_setting(tmp_path, capsys):
    assert main(["simulate", "--sx", "4", "--model", "x.txt", "--out", "y.txt"]) == 2
    assert "missing grid setting" in capsys.readouterr().err


@pytest.mark.gpu
def test_simulate_zero_model(tmp_path):
    model, out = str(tmp_path / "m.txt"), str(tmp_path / "d.txt")
    B.write_vector(np.zeros(GRID.n), model)
    assert main(["simulate", *GRID_FLAGS, "--model", model, "--out", out]) == 0
    assert np.all(B.read_vector(out) == 0.0)


@pytest.mark.gpu
def test_simulate_single_prism_matches_dense_column(tmp_path):
    model, out = str(tmp_path / "m.bin"), str(tmp_path / "d.bin")
    col = 17
    e = np.zeros(GRID.n)
    e[col] = 1.0
    B.write_vector(e, model)
    assert main(["simulate", *GRID_FLAGS, "--kernel", "magnetic", "--D", "33", "--I", "47",
                 "--F", "45000", "--model", model, "--out", out]) == 0
    og = O.ogrid(4, 3, 2, 1, 0, 0, 1, 1.0, 1.5, (0.0, 1.0, 2.5))
    ref = np.hstack(O.dense_layers(og, "magnetic", O.mag_constants(33.0, 47.0, 45000.0)))[:, col]
    assert np.linalg.norm(B.read_vector(out) - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.gpu
def test_gamma_scale_scales_output(tmp_path):
    model, o1, o2 = str(tmp_path / "m.txt"), str(tmp_path / "d1.txt"), str(tmp_path / "d2.txt")
    B.write_vector(np.ones(GRID.n), model)
    assert main(["simulate", *GRID_FLAGS, "--model", model, "--out", o1]) == 0
    assert main(["simulate", *GRID_FLAGS, "--gamma-scale", "1e5", "--model", model, "--out", o2]) == 0
    np.testing.assert_allclose(B.read_vector(o2), 1e5 * B.read_vector(o1), rtol=1e-12)


@pytest.mark.gpu
def test_length_mismatch_names_factorization(tmp_path, capsys):
    model, out = str(tmp_path / "m.txt"), str(tmp_path / "d.txt")
    B.write_vector(np.zeros(GRID.n + 1), model)
    assert main(["simulate", *GRID_FLAGS, "--model", model, "--out", out]) == 2
    err = capsys.readouterr().err
    assert f"n={GRID.n}" in err and f"{GRID.nx}*{GRID.ny}*{GRID.nz}" in err


@pytest.mark.gpu
def test_config_file_and_flag_override(tmp_path):
    cfg = tmp_path / "survey.cfg"
    cfg.write_text("# survey\nsx = 4\nsy = 3\nnz = 2\npxl = 1\npyr = 1\n"
                   "dx = 1.0\ndy = 9.9\nzblocks = 0,1,2.5\nkernel = gravity\n")
    model, out = str(tmp_path / "m.txt"), str(tmp_path / "d.txt")
    B.write_vector(np.zeros(GRID.n), model)
    assert main(["simulate", "--config", str(cfg), "--dy", "1.5", "--model", model, "--out", out]) == 0
    assert B.read_vector(out).shape == (GRID.m,)


@pytest.mark.gpu
def test_build_stack_then_apply_bit_identical(tmp_path):
    path, vec, out = str(tmp_path / "g.bttb"), str(tmp_path / "u.bin"), str(tmp_path / "d.bin")
    assert main(["build-stack", *GRID_FLAGS, "--out", path]) == 0
    rng = np.random.default_rng(10)
    u = rng.uniform(size=GRID.n)
    B.write_vector(u, vec)
    assert main(["apply", "--stack", path, "--in", vec, "--mode", "forward", "--out", out]) == 0
    with B.build_transform_stack(GRID, B.KernelParams.gravity()) as st:
        np.testing.assert_array_equal(B.read_vector(out), B.apply(st, u, "forward"))
        v = rng.uniform(size=GRID.m)
        B.write_vector(v, vec)
        assert main(["apply", "--stack", path, "--in", vec, "--mode", "transpose", "--out", out]) == 0
        np.testing.assert_array_equal(B.read_vector(out), B.apply(st, v, "transpose"))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("params", [B.KernelParams.gravity(), B.KernelParams.magnetic(33.0, 47.0, 45000.0)],
                         ids=["gravity", "magnetic"])
def test_persistence_round_trip_bit_identical(tmp_path, dtype, params):
    g = B.make_grid(7, 5, 3, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0))
    path = str(tmp_path / "s.bttb")
    rng = np.random.default_rng(88)
    u = rng.uniform(size=g.n)
    v = rng.uniform(size=g.m)
    with B.build_transform_stack(g, params, dtype=dtype) as st:
        B.save_stack(st, path)
        f0, t0 = B.apply(st, u, "forward"), B.apply(st, v, "transpose")
    with B.load_stack(path) as ld:
        assert ld.kind == params.kind and ld.grid == g and ld.dtype == np.dtype(dtype)
        np.testing.assert_array_equal(B.apply(ld, u, "forward"), f0)
        np.testing.assert_array_equal(B.apply(ld, v, "transpose"), t0)


@pytest.mark.gpu
def test_persistence_layer_shard(tmp_path):
    g = B.make_grid(6, 5, 4, 1, 1, 1, 1, 1.0, 1.5, (0.0, 1.0, 2.5, 3.0, 4.0))
    p = B.KernelParams.magnetic(10.0, 60.0, 50000.0)
    path = str(tmp_path / "shard.bttb")
    x = np.random.default_rng(3).uniform(size=2 * g.n_r)
    with B.build_transform_stack(g, p, layers=(1, 3)) as st:
        B.save_stack(st, path)
        f0 = B.apply(st, x, "forward")
    with B.load_stack(path) as ld:
        assert (ld.layer_begin, ld.layer_end) == (1, 3)
        np.testing.assert_array_equal(B.apply(ld, x, "forward"), f0)


def test_bad_magic_and_reference_format(tmp_path):
    junk = tmp_path / "junk.bttb"
    junk.write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(ValueError, match="magic"):
        B.load_stack(str(junk))
    ref = tmp_path / "ref.bttb"
    ref.write_bytes(b"BTTB" + b"\0" * 64)
    with pytest.raises(ValueError, match="unsupported stack version 0"):
        B.load_stack(str(ref))


REF_FILES = {"gravity": "ref_stack_gravity.bttb", "magnetic": "ref_stack_magnetic.bttb"}
REF_KEYS = {"gravity": "gravity_2_1_1_2", "magnetic": "magnetic_2_1_1_2"}


def _golden_path(name):
    from conftest import GOLDEN
    return os.path.join(GOLDEN, name)


@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_reference_file_truncated_or_inconsistent(tmp_path, kind):
    """Reference-format errors are raised while parsing (no GPU needed)."""
    data = open(_golden_path(REF_FILES[kind]), "rb").read()
    cut = tmp_path / "cut.bttb"
    cut.write_bytes(data[:-8])
    with pytest.raises(ValueError, match="truncated"):
        B.load_stack(str(cut))
    # header (magic 4 + version/kind 5 + 7 counts 56 + spacings 16 + 3 depths 24) then layer count
    off = 4 + 5 + 56 + 16 + 24
    bad = bytearray(data)
    bad[off:off + 8] = (5).to_bytes(8, "little")
    badp = tmp_path / "bad.bttb"
    badp.write_bytes(bytes(bad))
    with pytest.raises(ValueError, match="inconsistent"):
        B.load_stack(str(badp))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_load_reference_format_file(golden, kind, dtype):
    """A stack file written by the REFERENCE's save_stack loads and reproduces
    the reference's own products (tests/golden/make_golden.py stack_files)."""
    z = golden("small_6x5x2.npz")
    key = REF_KEYS[kind]
    u, v = z[f"{key}/u"], z[f"{key}/v"]
    tol = 1e-12 if dtype == "float64" else 1e-5
    with B.load_stack(_golden_path(REF_FILES[kind]), dtype=dtype) as st:
        assert st.kind == kind and st.dtype == np.dtype(dtype) and st.params is None
        assert st.grid == B.make_grid(6, 5, 2, 2, 1, 1, 2, 1.0, 1.5, (0.0, 1.0, 2.5))
        uq = u.astype(dtype).astype(float)
        vq = v.astype(dtype).astype(float)
        g = O.ogrid(6, 5, 2, 2, 1, 1, 2, 1.0, 1.5, (0.0, 1.0, 2.5))
        fw, tr = O.build_spectra(g, kind, O.grav_constants() if kind == "gravity"
                                 else O.mag_constants(33.0, 47.0, 45000.0))
        ref_f = z[f"{key}/fwd"] if dtype == "float64" else O.forward(g, fw, uq)
        ref_t = z[f"{key}/tra"] if dtype == "float64" else O.transpose(g, tr, vq)
        assert O.rel_l2(ref_f, B.apply(st, u, "forward")) <= tol
        assert O.rel_l2(ref_t, B.apply(st, v, "transpose")) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("params", [B.KernelParams.gravity(), B.KernelParams.magnetic(33.0, 47.0, 45000.0)],
                         ids=["gravity", "magnetic"])
def test_save_reference_format_and_lazy_spectra(tmp_path, params):
    """save_stack(format="reference") writes the reference layout: its arrays
    equal the oracle's fft2(T^circ) / fft2(transpose layout); the lazy
    TransformStack.forward/.transpose are the same arrays; the file loads back."""
    g = B.make_grid(7, 5, 3, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0))
    og = O.ogrid(7, 5, 3, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0))
    consts = O.grav_constants() if params.kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    fw, tr = O.build_spectra(og, params.kind, consts)
    path = str(tmp_path / "ref.bttb")
    rng = np.random.default_rng(8)
    u, v = rng.uniform(size=g.n), rng.uniform(size=g.m)
    with B.build_transform_stack(g, params) as st:
        assert len(st.forward) == g.nz and sum(a.size for a in st.forward) == st.element_count
        for r in range(g.nz):
            scale = np.abs(fw[r]).max()
            assert np.abs(st.forward[r] - fw[r]).max() <= 1e-13 * scale
            assert np.abs(st.transpose[r] - tr[r]).max() <= 1e-13 * scale
        B.save_stack(st, path, format="reference")
        f0, t0 = B.apply(st, u, "forward"), B.apply(st, v, "transpose")
    mx, my = g.embed_shape
    raw = open(path, "rb").read()
    assert raw[:4] == b"BTTB"
    head = 4 + 5 + 56 + 16 + 8 * (g.nz + 1) + 24
    arrs = np.frombuffer(raw[head:], dtype="<c16").reshape(2, g.nz, mx, my)
    for r in range(g.nz):
        scale = np.abs(fw[r]).max()
        assert np.abs(arrs[0, r] - fw[r]).max() <= 1e-13 * scale
        assert np.abs(arrs[1, r] - tr[r]).max() <= 1e-13 * scale
    with B.load_stack(path) as ld:
        assert O.rel_l2(f0, B.apply(ld, u, "forward")) <= 1e-13
        assert O.rel_l2(t0, B.apply(ld, v, "transpose")) <= 1e-13


@pytest.mark.gpu
def test_save_reference_format_needs_every_layer(tmp_path):
    g = B.make_grid(6, 5, 4, 1, 1, 1, 1, 1.0, 1.5, (0.0, 1.0, 2.5, 3.0, 4.0))
    with B.build_transform_stack(g, B.KernelParams.gravity(), layers=(1, 3)) as st:
        with pytest.raises(ValueError, match="every layer"):
            B.save_stack(st, str(tmp_path / "x.bttb"), format="reference")


@pytest.mark.gpu
def test_truncated_stack(tmp_path):
    g = B.make_grid(3, 2, 1, 0, 0, 0, 0, 1.0, 1.0, (0.0, 1.0))
    path = tmp_path / "s.bttb"
    with B.build_transform_stack(g, B.KernelParams.gravity()) as st:
        B.save_stack(st, str(path))
    data = path.read_bytes()
    path.write_bytes(data[:-8])
    with pytest.raises(ValueError, match="truncated"):
        B.load_stack(str(path))


@pytest.mark.gpu
def test_cli_reference_format_round_trip(tmp_path):
    path, vec, out = str(tmp_path / "r.bttb"), str(tmp_path / "u.bin"), str(tmp_path / "d.bin")
    assert main(["build-stack", *GRID_FLAGS, "--format", "reference", "--out", path]) == 0
    assert open(path, "rb").read(4) == b"BTTB"
    u = np.random.default_rng(12).uniform(size=GRID.n)
    B.write_vector(u, vec)
    assert main(["apply", "--stack", path, "--in", vec, "--mode", "forward", "--out", out]) == 0
    with B.build_transform_stack(GRID, B.KernelParams.gravity()) as st:
        assert O.rel_l2(B.apply(st, u, "forward"), B.read_vector(out)) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_loaded_stack_exposes_file_spectra(tmp_path, kind):
    """A loaded stack has no kernel constants; its lazy reference-shaped
    spectra come from the cached device spectra, so they equal the file's
    arrays (reference format) / the saving plan's (native format), and
    re-saving in the reference layout reproduces the file."""
    raw = open(_golden_path(REF_FILES[kind]), "rb").read()
    g = B.make_grid(6, 5, 2, 2, 1, 1, 2, 1.0, 1.5, (0.0, 1.0, 2.5))
    mx, my = g.embed_shape
    head = 4 + 5 + 56 + 16 + 8 * (g.nz + 1) + 24
    arrs = np.frombuffer(raw[head:], dtype="<c16").reshape(2, g.nz, mx, my)
    with B.load_stack(_golden_path(REF_FILES[kind])) as ld:
        for r in range(g.nz):
            scale = np.abs(arrs[0, r]).max()
            assert np.abs(ld.forward[r] - arrs[0, r]).max() <= 1e-13 * scale
            assert np.abs(ld.transpose[r] - arrs[1, r]).max() <= 1e-13 * scale
        path = str(tmp_path / "native.bttb")
        B.save_stack(ld, path)
        again = str(tmp_path / "again.bttb")
        B.save_stack(ld, again, format="reference")
    back = np.frombuffer(open(again, "rb").read()[head:], dtype="<c16").reshape(2, g.nz, mx, my)
    assert np.abs(back - arrs).max() <= 1e-13 * np.abs(arrs).max()
    with B.load_stack(path) as nat:
        for r in range(g.nz):
            assert np.abs(nat.forward[r] - arrs[0, r]).max() <= 1e-13 * np.abs(arrs[0, r]).max()
