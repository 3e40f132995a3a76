"""Layer-sharded operator across 2 processes (gloo, CPU) equals the unsharded one.

The multi-GPU path (paper_1912_06976_b200/parallel.py) shards contiguous
depth-layer blocks: forward partials are all-reduced, the data vector is
broadcast for the transpose.  Here the per-rank local operator is the CPU
oracle so the host-side sharding logic is exercised without GPUs; on B200s
the same ShardedOperator wraps DeviceOperator over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bttb_oracle as O
from paper_1912_06976_b200.parallel import ShardedOperator, partition_layers


class OracleLocal:
    """CPU stand-in for DeviceOperator over layers [lo, hi)."""

    def __init__(self, g, kind, consts, lo, hi):
        self.g = g
        self.layers = list(range(lo, hi))
        self.fw, self.tr = O.build_spectra(g, kind, consts, self.layers)

    def forward(self, x_local):
        return torch.from_numpy(O.forward(self.g, self.fw, x_local.numpy(), layers=self.layers))

    def transpose(self, d):
        return torch.from_numpy(O.transpose(self.g, self.tr, d.numpy()))


def _worker(rank, world, port, kind, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = O.ogrid(7, 5, 5, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0, 4.5, 6.0))
    consts = O.grav_constants() if kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    lo, hi = partition_layers(g.nz, world)[rank]
    op = ShardedOperator(OracleLocal(g, kind, consts, lo, hi))
    rng = np.random.default_rng(3)
    x = rng.uniform(size=g.n)
    v = rng.uniform(size=g.m)
    d = op.forward(torch.from_numpy(x[lo * g.n_r:hi * g.n_r].copy()))
    # rank 0 owns the data vector; other ranks pass garbage that the broadcast overwrites
    vt = torch.from_numpy(v.copy()) if rank == 0 else torch.zeros(g.m, dtype=torch.float64)
    xt = op.transpose(vt)
    parts = [torch.zeros(0, dtype=torch.float64)] * world
    dist.all_gather_object(parts, xt.numpy())
    if rank == 0:
        out["d"] = d.numpy().copy()
        out["xt"] = np.concatenate(parts)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_two_rank_layer_sharding_matches_unsharded(kind):
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), kind, out), nprocs=world, join=True)
        d, xt = out["d"], out["xt"]
    g = O.ogrid(7, 5, 5, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0, 4.5, 6.0))
    consts = O.grav_constants() if kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    fw, tr = O.build_spectra(g, kind, consts)
    rng = np.random.default_rng(3)
    x = rng.uniform(size=g.n)
    v = rng.uniform(size=g.m)
    assert O.rel_l2(O.forward(g, fw, x), d) <= 1e-14
    assert np.array_equal(O.transpose(g, tr, v), xt)
