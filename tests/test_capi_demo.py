"""The C ABI from plain C (examples/capi_demo.c): compiled with the system C
compiler against include/ and the built library, run on the GPU, and its
forward / transpose outputs compared with the Python mirror (same plan,
same inputs) and with the adjoint identity it checks itself."""
import os
import shutil
import subprocess

import numpy as np
import pytest

import paper_1912_06976_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1912_06976_b200")


def _compile(tmp_path):
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "capi_demo")
    subprocess.run([cc, "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "capi_demo.c"),
                    "-L", PKG, "-lbttb_sm100", f"-Wl,-rpath,{PKG}", "-lm", "-o", exe], check=True)
    return exe


def test_capi_demo_compiles(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_capi_demo_matches_python_mirror(tmp_path):
    exe = _compile(tmp_path)
    params = B.KernelParams.magnetic(33.0, 47.0, 45000.0)
    r = subprocess.run([exe] + [repr(float(c)) for c in params.gc], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout[-500:]
    lines = {ln.split()[0]: ln.split()[1:] for ln in r.stdout.splitlines()}
    fwd = np.array(lines["forward"], dtype=float)
    tra = np.array(lines["transpose"], dtype=float)
    g = B.make_grid(6, 5, 2, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5))
    x = np.sin(np.arange(g.n, dtype=float))
    v = np.cos(np.arange(g.m, dtype=float))
    with B.build_transform_stack(g, params) as st:
        np.testing.assert_array_equal(fwd, B.apply(st, x, "forward"))
        np.testing.assert_array_equal(tra, B.apply(st, v, "transpose"))
