"""The C-ABI library loads and exports every symbol include/bttb_sm100.h declares.

CPU only: no compute call is made except those that must fail loudly without
a GPU (the product path has no CPU fallback).
"""
import ctypes
import os
import re

import pytest

from paper_1912_06976_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "bttb_sm100.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(bttb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_exports():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_and_length_family():
    lib = _lib.lib()
    assert b"sm_100a" in lib.bttb_version()
    # smallest supported FFT length >= n: 2^a (a>=3), 2^a*3^b or 2^a*5^b (a>=2, b>=1),
    # or a power of two with a compile-time plan within 5% of it (2048); above
    # 8192 the generic-length path: the smallest 2^a 3^b 5^c (at most 65536)
    expect = {1: 8, 3: 8, 9: 12, 11: 12, 13: 16, 49: 64, 79: 80, 99: 100, 335: 384, 419: 432,
              511: 512, 1999: 2048, 1990: 2048, 1900: 1944, 2049: 2304, 8192: 8192, 8193: 8640,
              8599: 8640, 9000: 9000, 16385: 16875, 65536: 65536, 65537: -1}
    for n, L in expect.items():
        assert lib.bttb_fft_length(n) == L, n


def test_invalid_arguments_are_reported_with_messages():
    lib = _lib.lib()
    z = (ctypes.c_double * 3)(0.0, 1.0, 2.0)
    g = _lib.BttbGrid(4, 3, 2, 0, 0, 0, 0, 1.0, 1.0, ctypes.cast(z, ctypes.POINTER(ctypes.c_double)))
    k = _lib.BttbKernel()
    k.kind = _lib.GRAVITY
    k.gamma_scaled = 6.6743e-11
    h = ctypes.c_void_p()
    rc = lib.bttb_plan_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(k), 7, 0, 0, 2, 0, 0)
    assert rc == _lib.BTTB_EINVAL and "dtype" in _lib.last_error()
    rc = lib.bttb_plan_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(k), 0, 0, 1, 1, 0, 0)
    assert rc == _lib.BTTB_EINVAL and "layer range" in _lib.last_error()
    z2 = (ctypes.c_double * 3)(0.0, 2.0, 1.0)
    g.z_blocks = ctypes.cast(z2, ctypes.POINTER(ctypes.c_double))
    rc = lib.bttb_plan_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(k), 0, 0, 0, 2, 0, 0)
    assert rc == _lib.BTTB_EINVAL and "z2 >= z1" in _lib.last_error()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly_no_cpu_fallback():
    import paper_1912_06976_b200 as B
    g = B.make_grid(4, 3, 2, 0, 0, 0, 0, 1.0, 1.0, (0.0, 1.0, 2.0))
    with pytest.raises(B.CudaError, match="CUDA"):
        B.build_transform_stack(g, B.KernelParams.gravity())
    t = B.sym_distances(g)
    with pytest.raises(B.CudaError):
        B.gravity_layer_response(0.5, 1.5, t, B.KernelParams.gravity())
