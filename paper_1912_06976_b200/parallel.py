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

__all__ = ["partition_layers", "DeviceOperator", "ShardedOperator", "sharded_cgls"]


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
    """Device-resident local operator over a TransformStack (no host copies).

    Every tensor handed to the C ABI is checked first (dtype, device,
    contiguity, trailing length): the library takes raw pointers, so a
    float64 tensor on an fp32 plan or a strided layer slice would otherwise
    be read or written out of bounds (parallel.py:62).
    """

    def __init__(self, stack):
        from .multiply import apply_into

        self.stack = stack
        self._apply = apply_into
        self.dtype = torch.float64 if stack.dtype.itemsize == 8 else torch.float32
        self.device = torch.device("cuda", stack.device)

    def _check(self, t, last, what, dims=1):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{what} must be a torch tensor")
        if t.dtype != self.dtype:
            raise ValueError(f"{what} has dtype {t.dtype}, the plan computes in {self.dtype}")
        if t.device != self.device:
            raise ValueError(f"{what} lives on {t.device}, the plan on {self.device}")
        if not t.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if t.dim() < dims or tuple(t.shape[-dims:]) != tuple(last):
            raise ValueError(f"{what} must end in {tuple(last)}, got {tuple(t.shape)}")

    def _out(self, out, lead, last, like, what):
        if out is None:
            return torch.empty(tuple(lead) + tuple(last), dtype=self.dtype, device=like.device)
        self._check(out, last, what, len(last))
        if tuple(out.shape[:-len(last)]) != tuple(lead):
            raise ValueError(f"{what} has leading shape {tuple(out.shape[:-len(last)])}, "
                             f"expected {tuple(lead)}")
        return out

    def forward(self, x_local, out=None):
        g = self.stack.grid
        self._check(x_local, (self.stack.n_local,), "x_local")
        batch = 1 if x_local.dim() == 1 else x_local.shape[0]
        out = self._out(out, x_local.shape[:-1], (g.m,), x_local, "out")
        self._apply(self.stack, "forward", x_local.data_ptr(), out.data_ptr(), batch,
                    torch.cuda.current_stream(x_local.device).cuda_stream)
        return out

    def transpose(self, d, out=None):
        self._check(d, (self.stack.grid.m,), "d")
        batch = 1 if d.dim() == 1 else d.shape[0]
        out = self._out(out, d.shape[:-1], (self.stack.n_local,), d, "out")
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

        x_local = x_local.contiguous()
        self._check(x_local, (self.stack.n_local,), "x_local")
        out = torch.empty(self.spectrum_shape(x_local.shape[:-1]), dtype=self.dtype, device=x_local.device)
        return self._staged("forward", _lib.STAGE_TO_SPECTRUM, x_local, out)

    def from_spectrum(self, w, out=None):
        from . import _lib

        w = w.contiguous()
        self._check(w, self.spectrum_shape(), "w", 3)
        out = self._out(out, w.shape[:-3], (self.stack.grid.m,), w, "out")
        return self._staged("forward", _lib.STAGE_FROM_SPECTRUM, w, out)

    def transpose_spectrum(self, d):
        from . import _lib

        d = d.contiguous()
        self._check(d, (self.stack.grid.m,), "d")
        out = torch.empty(self.spectrum_shape(d.shape[:-1]), dtype=self.dtype, device=d.device)
        return self._staged("transpose", _lib.STAGE_TO_SPECTRUM, d, out)

    def transpose_from_spectrum(self, w, out=None):
        from . import _lib

        w = w.contiguous()
        self._check(w, self.spectrum_shape(), "w", 3)
        out = self._out(out, w.shape[:-3], (self.stack.n_local,), w, "out")
        return self._staged("transpose", _lib.STAGE_FROM_SPECTRUM, w, out)


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

    def _root(self):
        """Global rank of the group's rank 0 (broadcast's ``src`` is global;
        ADVICE r1: parallel.py:157)."""
        return 0 if self.group is None else dist.get_global_rank(self.group, 0)

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
                dist.broadcast(w, src=self._root(), group=self.group)
            return self.local.transpose_from_spectrum(w, out) if out is not None else \
                self.local.transpose_from_spectrum(w)
        if self._multi():
            dist.broadcast(d, src=self._root(), group=self.group)
        return self.local.transpose(d, out) if out is not None else self.local.transpose(d)


def sharded_cgls(op, d, iters=10, damp=0.0, rtol=1e-13, history=True):
    """Layer-sharded CGLS (BASELINE configs[4]: "layers sharded" at 1/2/4/8 GPUs).

    ``op`` is a :class:`ShardedOperator`; each rank holds its layer block of
    the models m, p and s (the same contiguous blocks ``partition_layers``
    gives the spectrum caches), and the data-space vectors d, r, q are
    replicated.  Per iteration: the local forward partial G_k p_k, ONE
    all-reduce of it (the reference's layer sum, multiply.py:42-45, split
    across ranks -- SPEC.md:316 notes the reduction), the local transpose of
    the replicated residual (no broadcast needed: every rank holds the same
    r), and two all-reduces of per-model fp64 scalars (|p|^2 for the damping
    term, |s|^2).  The recurrences, the fp64 dot products and the freeze rule
    (alpha = beta = 0 once |s_k| <= rtol |s_0|) are those of the single-GPU
    loop (``bttb_cgls``) and of the oracle's ``cgls``.

    d: (m,) or (batch, m) tensor (the root's copy is broadcast first).
    Returns (m_local, hist): this rank's layer block of the models, shaped
    like d with the last axis n_local, and the residual norms |r_k|,
    k = 0..iters, as a (batch, iters+1) float64 tensor on d's device (or None).
    """
    if int(iters) != iters or iters < 0:
        raise ValueError(f"iters must be a non-negative integer, got {iters!r}")
    local, grp = op.local, op.group
    multi = op._multi()

    def allsum(t):
        if multi:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=grp)
        return t

    def dot(a):  # per-model fp64 sum of squares over the last axis
        return (a.to(torch.float64) ** 2).sum(-1)

    if multi:
        d = d.contiguous()
        dist.broadcast(d, src=op._root(), group=grp)
    dd = float(damp) * float(damp)
    r = d.clone()
    s = local.transpose(r)
    m = torch.zeros_like(s)
    p = s.clone()
    gamma = allsum(dot(s))
    floor = rtol * rtol * gamma
    hist = [dot(r).sqrt()] if history else None
    for _ in range(int(iters)):
        q = allsum(local.forward(p))
        delta = dot(q)
        if dd:
            delta = delta + dd * allsum(dot(p))
        live = gamma > floor
        alpha = torch.where((delta > 0) & live, gamma / torch.where(delta > 0, delta, torch.ones_like(delta)),
                            torch.zeros_like(gamma))
        a_ = alpha.to(s.dtype).unsqueeze(-1)
        m = m + a_ * p
        r = r - a_ * q
        s = local.transpose(r)
        if dd:
            s = s - dd * m
        gnew = allsum(dot(s))
        beta = torch.where(live, gnew / torch.where(live, gamma, torch.ones_like(gamma)), torch.zeros_like(gamma))
        gamma = gnew
        p = s + beta.to(s.dtype).unsqueeze(-1) * p
        if history:
            hist.append(dot(r).sqrt())
    if history:
        hist = torch.stack(hist, dim=-1)
        if hist.dim() == 1:
            hist = hist.unsqueeze(0)
    return m, hist
