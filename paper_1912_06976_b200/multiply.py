"""Forward and transpose products through the device spectrum cache.

Drop-in for ``/root/reference/pkg/src/bttb/multiply.py``: same ``apply(stack,
x, mode)`` signature, vector ordering, ValueError messages and a NEW returned
array (x is never mutated).  Extensions: a leading batch axis, and CUDA torch
tensors in/out (zero-copy device pointers on the current stream) for
device-resident iterative use.
"""
import numpy as np

from . import _lib

__all__ = ["apply", "relative_error"]

# Host buffers of the numpy path.  A freshly allocated pageable destination
# page-faults under the device-to-host copy (C4 model, 1.03 GB: 203 ms on a
# B200 box, vs 18 ms into pinned memory -- tools/hostcopy_probe.py), so large
# outputs are allocated in pinned memory (torch's caching host allocator: the
# pages are reused across calls and live as long as the returned array).
# Large pageable INPUTS are handled by the library (csrc/hoststage.cu:
# chunked staging through a pinned ring by a pool of host threads, overlapped
# with the copy engine).
_PINNED_MIN = 1 << 22


def _pinned_empty(shape, dt):
    try:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError
        t = torch.empty(tuple(shape), dtype=torch.float64 if dt == np.float64 else torch.float32, pin_memory=True)
    except Exception:  # no torch / no CUDA runtime: the library stages the copy itself
        return np.empty(shape, dtype=dt)
    return t.numpy()


def _host_in(xa, dt):
    """x as a contiguous `dt` array (the library stages pageable memory)."""
    return np.ascontiguousarray(xa, dtype=dt)


def _host_out(shape, dt):
    nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
    return _pinned_empty(shape, dt) if nbytes >= _PINNED_MIN else np.empty(shape, dtype=dt)

_MODES = {"forward": _lib.FORWARD, "transpose": _lib.TRANSPOSE}


def _expected(stack, mode):
    g = stack.grid
    if mode == "forward":
        return stack.n_local, (f"forward expects a vector of length n={stack.n_local} "
                               f"= nx*ny*nz = {g.nx}*{g.ny}*{stack.nz_local}")
    return g.m, f"transpose expects a vector of length m={g.m}"


def _is_torch(x):
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


def apply(stack, x, mode, stream=None):
    """Multiply by the operator (``"forward"``: d = G m) or its transpose.

    x: (n,) / (batch, n) model vectors for forward, (m,) / (batch, m) data
    vectors for transpose (multiply.py:22-58).  numpy input runs host-to-host
    through the C ABI and returns a new float64 (fp32 plan: float32) array;
    a CUDA torch tensor runs device-to-device on ``stream`` (default: the
    current torch stream) and returns a new tensor; with an explicit stream
    the work is ordered after the current stream and the current stream is
    ordered after the result, so the tensor is safe to use on either.
    """
    if mode not in _MODES:
        raise ValueError(f"mode must be 'forward' or 'transpose', got {mode!r}")
    want, msg = _expected(stack, mode)
    other = stack.grid.m if mode == "forward" else stack.n_local
    if _is_torch(x):
        return _apply_torch(stack, x, mode, want, other, msg, stream)
    dt = stack.dtype
    xa = np.asarray(x, dtype=float)
    if xa.ndim not in (1, 2) or xa.shape[-1] != want:
        raise ValueError(f"{msg}, got shape {xa.shape}")
    batch = 1 if xa.ndim == 1 else xa.shape[0]
    xin = _host_in(xa, dt)
    out = _host_out(xa.shape[:-1] + (other,), dt)
    _lib.check(_lib.lib().bttb_apply(stack.handle, _MODES[mode],
                                     xin.ctypes.data_as(_lib.ctypes.c_void_p),
                                     out.ctypes.data_as(_lib.ctypes.c_void_p),
                                     batch, _lib.HOST_PTR, None))
    return out


def _apply_torch(stack, x, mode, want, other, msg, stream):
    import torch

    if not x.is_cuda:
        raise ValueError("torch tensors must live on a CUDA device")
    if x.dim() not in (1, 2) or x.shape[-1] != want:
        raise ValueError(f"{msg}, got shape {tuple(x.shape)}")
    tdt = torch.float64 if stack.dtype == np.float64 else torch.float32
    xin = x.to(dtype=tdt).contiguous()
    out = torch.empty(tuple(x.shape[:-1]) + (other,), dtype=tdt, device=x.device)
    batch = 1 if x.dim() == 1 else x.shape[0]
    cur = torch.cuda.current_stream(x.device)
    st = cur if stream is None else stream
    if st != cur:
        # xin / out are allocated (and xin possibly written) on the current
        # stream: order the library's work after it, keep both blocks alive
        # for `st` in the caching allocator, and order the caller's stream
        # after the result (multiply.py:64)
        st.wait_stream(cur)
        xin.record_stream(st)
        out.record_stream(st)
    _lib.check(_lib.lib().bttb_apply(stack.handle, _MODES[mode], _lib.ctypes.c_void_p(xin.data_ptr()),
                                     _lib.ctypes.c_void_p(out.data_ptr()), batch,
                                     _lib.DEVICE_PTR, _lib.ctypes.c_void_p(st.cuda_stream)))
    if st != cur:
        cur.wait_stream(st)
    return out


def apply_into(stack, mode, x_ptr, y_ptr, batch=1, stream_ptr=None, host=False):
    """Raw-pointer entry (bench / multi-GPU driver): y <- op(x), no validation copies.

    host=False: device pointers; host=True: host pointers, synchronous;
    host="async": pinned host pointers, returns at once -- the input copy is
    ordered after the work already queued on ``stream_ptr`` (default stream if
    None), x / y are in use until that stream is synchronised
    (BTTB_HOST_ASYNC); host="async-unordered": the same without the ordering
    edge (x must be final at call time), so consecutive calls overlap their
    copies (BTTB_HOST_ASYNC_UNORDERED)."""
    wheres = {False: _lib.DEVICE_PTR, True: _lib.HOST_PTR, "async": _lib.HOST_ASYNC,
              "async-unordered": _lib.HOST_ASYNC_UNORDERED}
    if host not in wheres:
        raise ValueError(f"host must be one of {sorted(map(str, wheres))}, got {host!r}")
    where = wheres[host]
    _lib.check(_lib.lib().bttb_apply(stack.handle, _MODES[mode], _lib.ctypes.c_void_p(x_ptr),
                                     _lib.ctypes.c_void_p(y_ptr), int(batch), where,
                                     _lib.ctypes.c_void_p(stream_ptr or 0)))


def relative_error(a, b):
    """||a - b|| / ||a||; 0 if both zero, inf if only a is (multiply.py:61-71)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    na = np.linalg.norm(a)
    diff = np.linalg.norm(a - b)
    if na == 0.0:
        return 0.0 if diff == 0.0 else np.inf
    return diff / na
