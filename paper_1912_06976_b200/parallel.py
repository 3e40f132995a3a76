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

The local operator is anything with ``forward(x_local) -> d`` and
``transpose(d) -> x_local`` on tensors; on GPUs it is :class:`DeviceOperator`
over a layer-range :class:`~paper_1912_06976_b200.transform.TransformStack`.
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


class ShardedOperator:
    """Layer-sharded G and G^T over a process group (NCCL on GPUs, gloo in tests)."""

    def __init__(self, local, group=None):
        self.local = local
        self.group = group

    def forward(self, x_local, out=None):
        d = self.local.forward(x_local, out) if out is not None else self.local.forward(x_local)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(d, op=dist.ReduceOp.SUM, group=self.group)
        return d

    def transpose(self, d, out=None):
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.broadcast(d, src=0, group=self.group)
        return self.local.transpose(d, out) if out is not None else self.local.transpose(d)
