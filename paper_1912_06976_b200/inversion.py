"""Device-resident batched CGLS on the fast operator.

The paper leaves a GPU inversion loop as future work and the
reference package stops at ``apply`` (multiply.py:22-58; inversion is a
non-goal).  ``cgls`` runs the whole loop inside the library
(``bttb_cgls``): one forward and one transpose product per iteration through
the cached spectra, fused vector updates, fp64 reductions, scalars kept on the
device -- no host round trip between iterations.
"""
import numpy as np

from . import _lib

__all__ = ["cgls", "cgls_into"]


def cgls(stack, d, iters=10, damp=0.0, stream=None, history=True):
    """Minimise |G m - d|^2 + damp^2 |m|^2 from m = 0 with ``iters`` CGLS steps.

    d: (m,) or (batch, m) data vectors -- numpy (host-to-host) or a CUDA torch
    tensor (device-resident, runs on ``stream``, default the current stream).
    Returns ``(models, resid)``: models shaped like d with the last axis n,
    and, if ``history``, the data-residual norms |d - G m_k|, k = 0..iters,
    shaped (iters+1,) or (batch, iters+1) (else None).  The stack must hold
    every layer (a layer-sharded stack needs the multi-GPU driver).
    """
    if int(iters) != iters or iters < 0:
        raise ValueError(f"iters must be a non-negative integer, got {iters!r}")
    if not np.isfinite(damp) or damp < 0:
        raise ValueError(f"damp must be finite and >= 0, got {damp!r}")
    g = stack.grid
    msg = f"cgls expects data of length m={g.m}"
    torch_in = type(d).__module__.startswith("torch") and hasattr(d, "data_ptr")
    if torch_in:
        import torch

        if not d.is_cuda:
            raise ValueError("torch tensors must live on a CUDA device")
        if d.dim() not in (1, 2) or d.shape[-1] != g.m:
            raise ValueError(f"{msg}, got shape {tuple(d.shape)}")
        tdt = torch.float64 if stack.dtype == np.float64 else torch.float32
        din = d.to(dtype=tdt).contiguous()
        batch = 1 if d.dim() == 1 else d.shape[0]
        out = torch.empty(tuple(d.shape[:-1]) + (stack.n_local,), dtype=tdt, device=d.device)
        cur = torch.cuda.current_stream(d.device)
        st = cur if stream is None else stream
        if st != cur:  # see multiply._apply_torch: order, keep alive, hand back
            st.wait_stream(cur)
            din.record_stream(st)
            out.record_stream(st)
        xp, yp, where, sp = din.data_ptr(), out.data_ptr(), _lib.DEVICE_PTR, st.cuda_stream
        shape = tuple(d.shape[:-1])
    else:
        da = np.asarray(d, dtype=float)
        if da.ndim not in (1, 2) or da.shape[-1] != g.m:
            raise ValueError(f"{msg}, got shape {da.shape}")
        batch = 1 if da.ndim == 1 else da.shape[0]
        from .multiply import _host_in, _host_out  # pinned host buffers for the copy engines

        din = _host_in(da, stack.dtype)
        out = _host_out(da.shape[:-1] + (stack.n_local,), stack.dtype)
        xp, yp, where, sp = din.ctypes.data, out.ctypes.data, _lib.HOST_PTR, 0
        shape = da.shape[:-1]
    hist = np.empty((batch, int(iters) + 1), dtype=np.float64) if history else None
    c = _lib.ctypes
    _lib.check(_lib.lib().bttb_cgls(stack.handle, c.c_void_p(xp), c.c_void_p(yp), int(batch), int(iters),
                                    float(damp), where, c.c_void_p(sp),
                                    _lib.as_dptr(hist) if history else None))
    if torch_in and st != cur:
        cur.wait_stream(st)
    if hist is not None:
        hist = hist.reshape(shape + (int(iters) + 1,))
    return out, hist


def cgls_into(stack, d_ptr, m_ptr, batch, iters, damp=0.0, stream_ptr=None, host=False):
    """Raw-pointer entry (bench): m <- CGLS(d), device pointers or (host=True)
    host pointers -- pinned for full copy bandwidth -- with a synchronous return."""
    c = _lib.ctypes
    _lib.check(_lib.lib().bttb_cgls(stack.handle, c.c_void_p(d_ptr), c.c_void_p(m_ptr), int(batch), int(iters),
                                    float(damp), _lib.HOST_PTR if host else _lib.DEVICE_PTR,
                                    c.c_void_p(stream_ptr or 0), None))
