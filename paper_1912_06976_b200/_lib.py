"""ctypes binding of the sm_100a C ABI (include/bttb_sm100.h).

The product path has no CPU fallback: if the in-tree ``libbttb_sm100.so`` is
missing or cannot be loaded, every compute entry point raises
:class:`NativeLibraryError`.  Build it with ``python -c "import
__graft_entry__ as g; g.build()"`` (or ``paper_1912_06976_b200/_build.py``).
"""
import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# BTTB_LIB_PATH: a development build variant (paper_1912_06976_b200/_build.py --variant)
LIB_PATH = os.environ.get("BTTB_LIB_PATH") or os.path.join(_HERE, "libbttb_sm100.so")

BTTB_OK, BTTB_EINVAL, BTTB_ECUDA, BTTB_ENONFINITE, BTTB_ENOMEM = 0, -1, -2, -3, -4
GRAVITY, MAGNETIC = 0, 1
F64, F32 = 0, 1
FORWARD, TRANSPOSE = 0, 1
DEVICE_PTR, HOST_PTR, HOST_ASYNC, HOST_ASYNC_UNORDERED = 0, 1, 2, 3
STAGE_ALL, STAGE_TO_SPECTRUM, STAGE_FROM_SPECTRUM = 0, 1, 2

#: every symbol include/bttb_sm100.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "bttb_plan_create", "bttb_plan_create_from_spectra", "bttb_plan_create_from_windows", "bttb_plan_destroy",
    "bttb_apply", "bttb_apply_staged", "bttb_cgls", "bttb_layer_window",
    "bttb_layer_spectrum", "bttb_plan_info", "bttb_gravity_response",
    "bttb_magnetic_response", "bttb_fft_length", "bttb_debug_check_guards", "bttb_last_error", "bttb_version",
)


class NativeLibraryError(RuntimeError):
    """The sm_100a library is unavailable (no CPU fallback exists)."""


class CudaError(RuntimeError):
    """A CUDA call inside the library failed."""


class BttbGrid(ctypes.Structure):
    _fields_ = [("sx", ctypes.c_int64), ("sy", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("pxl", ctypes.c_int64), ("pxr", ctypes.c_int64), ("pyl", ctypes.c_int64),
                ("pyr", ctypes.c_int64), ("dx", ctypes.c_double), ("dy", ctypes.c_double),
                ("z_blocks", ctypes.POINTER(ctypes.c_double))]


class BttbKernel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("gamma_scaled", ctypes.c_double),
                ("gc", ctypes.c_double * 5)]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    dp = ctypes.POINTER(ctypes.c_double)
    lib.bttb_plan_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(BttbGrid),
                                     ctypes.POINTER(BttbKernel), ctypes.c_int, ctypes.c_int,
                                     i64, i64, i64, i64]
    lib.bttb_plan_create_from_spectra.argtypes = [ctypes.POINTER(P), ctypes.POINTER(BttbGrid),
                                                  ctypes.POINTER(BttbKernel), ctypes.c_int, ctypes.c_int,
                                                  i64, i64, i64, i64, P]
    lib.bttb_plan_create_from_windows.argtypes = [ctypes.POINTER(P), ctypes.POINTER(BttbGrid),
                                                  ctypes.POINTER(BttbKernel), ctypes.c_int, ctypes.c_int,
                                                  i64, i64, i64, i64, dp]
    lib.bttb_plan_destroy.argtypes = [P]
    lib.bttb_apply.argtypes = [P, ctypes.c_int, P, P, i64, ctypes.c_int, P]
    lib.bttb_apply_staged.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P, i64, P]
    lib.bttb_cgls.argtypes = [P, P, P, i64, ctypes.c_int, ctypes.c_double, ctypes.c_int, P, dp]
    lib.bttb_layer_window.argtypes = [P, i64, dp]
    lib.bttb_layer_spectrum.argtypes = [P, i64, P]
    lib.bttb_plan_info.argtypes = [P, ctypes.POINTER(i64)]
    lib.bttb_gravity_response.argtypes = [dp, i64, dp, i64, dp, dp, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double, dp, ctypes.c_int]
    lib.bttb_magnetic_response.argtypes = [dp, i64, dp, i64, dp, ctypes.c_double,
                                           ctypes.c_double, dp, dp, ctypes.c_int]
    lib.bttb_debug_check_guards.argtypes = [P]
    lib.bttb_debug_check_guards.restype = ctypes.c_int
    lib.bttb_fft_length.argtypes = [i64]
    lib.bttb_fft_length.restype = i64
    lib.bttb_last_error.restype = ctypes.c_char_p
    lib.bttb_version.restype = ctypes.c_char_p
    for name in ("bttb_plan_create", "bttb_plan_create_from_spectra", "bttb_plan_create_from_windows",
                 "bttb_plan_destroy", "bttb_apply", "bttb_apply_staged", "bttb_cgls", "bttb_layer_window",
                 "bttb_layer_spectrum", "bttb_plan_info", "bttb_gravity_response",
                 "bttb_magnetic_response"):
        getattr(lib, name).restype = ctypes.c_int


def lib():
    """Load (once) and return the library; raise NativeLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing: build the sm_100a library first "
                    "(python paper_1912_06976_b200/_build.py); there is no CPU fallback")
            try:
                handle = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(handle)
            _lib = handle
    return _lib


def last_error():
    return lib().bttb_last_error().decode()


def check(rc):
    """Map a status code to the reference's exception types."""
    if rc == BTTB_OK:
        return
    msg = last_error()
    if rc == BTTB_EINVAL:
        raise ValueError(msg)
    if rc == BTTB_ENONFINITE:
        raise FloatingPointError(msg)
    if rc == BTTB_ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg)


def as_dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
