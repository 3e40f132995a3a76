"""Depth-layer sharding across GPUs (one process per GPU, torch.distributed/NCCL).

The operator is a sum over depth layers (forward) and a stack of per-layer
outputs (transpose) -- multiply.py:42-45 / :54-56 of the reference, which runs
the layer loop serially.  Sharding contiguous layer blocks across ranks:

* forward: every rank applies its own layers (a partial station vector) and
  the partials are summed with one NCCL all-reduce of the m-vector (the
  "cheap variant" of SURVEY.md 8(e): each rank has already run its own inverse
  FFT, so only sx*sy values cross NVLink instead of a (Hx, Ly) spectrum; the
  result is replicated, ready for the next transpose of a CGLS loop);
* transpose: the data vector is broadcast from rank 0 (m values) and every
  rank emits its own layers into its own slice -- no gather.

``reduce="spectrum"`` is the north-star contract (BASELINE.json): the
forward sums the ranks' partial station half spectra W (Hx x sy complex, the
column-inverse-transformed cross-layer sum, 16.4 MB at C4 fp64) with one NCCL
all-reduce and runs ONE row inverse transform on the sum; the transpose
broadcasts the data's half spectrum from rank 0 and every rank runs its own
layers' column stages from it (C ABI ``bttb_apply_staged``).  It moves twice
the bytes of the default and saves each rank one row transform of the
stations, so the default stays ``"data"``.

The local operator is anything with ``forward(x_local) -> d`` and
``transpose(d) -> x_local`` on tensors (plus ``forward_spectrum``,
``from_spectrum``, ``transpose_spectrum``, ``transpose_from_spectrum`` for
``reduce="spectrum"``); on GPUs it is :class:`DeviceOperator` over a
layer-range :class:`~paper_1912_06976_b200.transform.TransformStack`.
"""
import torch
import torch.distributed as dist

__all__ = ["partition_layers", "DeviceOperator", "ShardedOperator"]


def partition_layers(nz, world):
    """Contiguous balanced layer ranges; the first nz % world ranks get one more.

    e.g. nz=20, world=8 -> 3,3,3,3,2,2,2,2.
    """
    if world < 1 or nz < world:
        raise ValueError(f"cannot shard {nz} layers over {world} ranks")
    base, extra = divmod(nz, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class DeviceOperator:
    """Device-resident local operator over a TransformStack (no host copies)."""

    def __init__(self, stack):
        from .multiply import apply_into

        self.stack = stack
        self._apply = apply_into
        self.dtype = torch.float64 if stack.dtype.itemsize == 8 else torch.float32

    def forward(self, x_local, out=None):
        g = self.stack.grid
        batch = 1 if x_local.dim() == 1 else x_local.shape[0]
        if out is None:
            out = torch.empty(x_local.shape[:-1] + (g.m,), dtype=self.dtype, device=x_local.device)
        self._apply(self.stack, "forward", x_local.data_ptr(), out.data_ptr(), batch,
                    torch.cuda.current_stream(x_local.device).cuda_stream)
        return out

    def transpose(self, d, out=None):
        batch = 1 if d.dim() == 1 else d.shape[0]
        if out is None:
            out = torch.empty(d.shape[:-1] + (self.stack.n_local,), dtype=self.dtype, device=d.device)
        self._apply(self.stack, "transpose", d.data_ptr(), out.data_ptr(), batch,
                    torch.cuda.current_stream(d.device).cuda_stream)
        return out

    # split products (reduce="spectrum"): W is (batch...,) + (Hx, sy, 2) reals
    def spectrum_shape(self, lead=()):
        lx, _ = self.stack.fft_shape
        return tuple(lead) + (lx // 2 + 1, self.stack.grid.sy, 2)

    def _staged(self, mode, stage, x, out):
        from . import _lib

        lead = x.shape[:-3] if stage == _lib.STAGE_FROM_SPECTRUM else x.shape[:-1]
        batch = 1
        for v in lead:
            batch *= v
        _lib.check(_lib.lib().bttb_apply_staged(
            self.stack.handle, _lib.FORWARD if mode == "forward" else _lib.TRANSPOSE, stage,
            _lib.ctypes.c_void_p(x.data_ptr()), _lib.ctypes.c_void_p(out.data_ptr()), batch,
            _lib.ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)))
        return out

    def empty_spectrum(self, lead, like):
        return torch.empty(self.spectrum_shape(lead), dtype=self.dtype, device=like.device)

    def forward_spectrum(self, x_local):
        from . import _lib

        out = torch.empty(self.spectrum_shape(x_local.shape[:-1]), dtype=self.dtype, device=x_local.device)
        return self._staged("forward", _lib.STAGE_TO_SPECTRUM, x_local.contiguous(), out)

    def from_spectrum(self, w, out=None):
        from . import _lib

        if out is None:
            out = torch.empty(w.shape[:-3] + (self.stack.grid.m,), dtype=self.dtype, device=w.device)
        return self._staged("forward", _lib.STAGE_FROM_SPECTRUM, w.contiguous(), out)

    def transpose_spectrum(self, d):
        from . import _lib

        out = torch.empty(self.spectrum_shape(d.shape[:-1]), dtype=self.dtype, device=d.device)
        return self._staged("transpose", _lib.STAGE_TO_SPECTRUM, d.contiguous(), out)

    def transpose_from_spectrum(self, w, out=None):
        from . import _lib

        if out is None:
            out = torch.empty(w.shape[:-3] + (self.stack.n_local,), dtype=self.dtype, device=w.device)
        return self._staged("transpose", _lib.STAGE_FROM_SPECTRUM, w.contiguous(), out)


class ShardedOperator:
    """Layer-sharded G and G^T over a process group (NCCL on GPUs, gloo in tests).

    reduce="data" (default): all-reduce of the ranks' partial station vectors;
    reduce="spectrum": all-reduce of the partial station half spectra, then one
    row inverse transform (see the module docstring)."""

    def __init__(self, local, group=None, reduce="data"):
        if reduce not in ("data", "spectrum"):
            raise ValueError(f"reduce must be 'data' or 'spectrum', got {reduce!r}")
        self.local = local
        self.group = group
        self.reduce = reduce

    def _multi(self):
        return dist.is_initialized() and dist.get_world_size(self.group) > 1

    def forward(self, x_local, out=None):
        if self.reduce == "spectrum":
            w = self.local.forward_spectrum(x_local)
            if self._multi():
                dist.all_reduce(w, op=dist.ReduceOp.SUM, group=self.group)
            return self.local.from_spectrum(w, out) if out is not None else self.local.from_spectrum(w)
        d = self.local.forward(x_local, out) if out is not None else self.local.forward(x_local)
        if self._multi():
            dist.all_reduce(d, op=dist.ReduceOp.SUM, group=self.group)
        return d

    def transpose(self, d, out=None):
        if self.reduce == "spectrum":
            rank = dist.get_rank(self.group) if self._multi() else 0
            if rank == 0:
                w = self.local.transpose_spectrum(d)
            else:
                w = self.local.empty_spectrum(d.shape[:-1], d)
            if self._multi():
                dist.broadcast(w, src=0, group=self.group)
            return self.local.transpose_from_spectrum(w, out) if out is not None else \
                self.local.transpose_from_spectrum(w)
        if self._multi():
            dist.broadcast(d, src=0, group=self.group)
        return self.local.transpose(d, out) if out is not None else self.local.transpose(d)
