"""The ctypes binding INTEGRATION.md section 3 shows a reference maintainer is
real code: it is executed here against the built library (argument
conversion on CPU; products against the package on a B200)."""
import ctypes
import os

import numpy as np
import pytest

import paper_1912_06976_b200 as B
from paper_1912_06976_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub():
    src = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = ""
    for start in ("# bttb/_gpu.py", "def cgls(h, d, n, iters"):
        blk = src[src.index(start):]
        code += blk[:blk.index("```")] + "\n"
    code = code.replace('ctypes.CDLL("libbttb_sm100.so")', f"ctypes.CDLL({_lib.LIB_PATH!r})")
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def _small():
    return B.make_grid(6, 5, 2, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5)), B.KernelParams.magnetic(33.0, 47.0, 45000.0)


def test_stub_signatures_convert():
    ns = _stub()
    assert ns["_lib"].bttb_apply.argtypes[2] is ctypes.c_void_p
    g, p = _small()
    try:
        ns["build"](g, p)
    except ValueError as exc:  # no GPU in the build container: a clean library error, not a ctypes one
        assert "device" in str(exc).lower() or "cuda" in str(exc).lower()


@pytest.mark.gpu
def test_stub_products_match_package():
    ns = _stub()
    g, p = _small()
    h = ns["build"](g, p)
    rng = np.random.default_rng(5)
    x, v = rng.uniform(size=g.n), rng.normal(size=g.m)
    with B.build_transform_stack(g, p) as st:
        np.testing.assert_array_equal(ns["apply"](h, x, "forward", g.m), B.apply(st, x, "forward"))
        np.testing.assert_array_equal(ns["apply"](h, v, "transpose", g.n), B.apply(st, v, "transpose"))
        m, hist = ns["cgls"](h, v, g.n, 4)
        m2, h2 = B.cgls(st, v, iters=4)
    np.testing.assert_array_equal(m, m2)
    np.testing.assert_array_equal(hist, h2)
    _lib.lib().bttb_plan_destroy(h)
