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

    # split products in the oracle's own spectral domain (full mx x my spectra,
    # multiply.py:42-45 / :52-56 split at the cross-layer sum), as real views
    def forward_spectrum(self, x_local):
        g, x = self.g, x_local.numpy()
        acc = np.zeros((g.mx, g.my), dtype=complex)
        for k in range(len(self.layers)):
            buf = np.zeros((g.mx, g.my))
            buf[:g.nx, :g.ny] = x[k * g.n_r:(k + 1) * g.n_r].reshape(g.ny, g.nx).T
            acc += self.fw[k] * np.fft.fft2(buf)
        return torch.view_as_real(torch.from_numpy(acc)).contiguous()

    def from_spectrum(self, w):
        g = self.g
        y = np.fft.ifft2(torch.view_as_complex(w.contiguous()).numpy())
        return torch.from_numpy(y.real[:g.sx, :g.sy].T.ravel().copy())

    def transpose_spectrum(self, d):
        g = self.g
        buf = np.zeros((g.mx, g.my))
        buf[:g.sx, :g.sy] = d.numpy().reshape(g.sy, g.sx).T
        return torch.view_as_real(torch.from_numpy(np.fft.fft2(buf))).contiguous()

    def empty_spectrum(self, lead, like):
        return torch.zeros(tuple(lead) + (self.g.mx, self.g.my, 2), dtype=torch.float64)

    def transpose_from_spectrum(self, w):
        g, vh = self.g, torch.view_as_complex(w.contiguous()).numpy()
        out = np.empty(len(self.tr) * g.n_r)
        for k, T in enumerate(self.tr):
            y = np.fft.ifft2(T * vh)
            out[k * g.n_r:(k + 1) * g.n_r] = y.real[:g.nx, :g.ny].T.ravel()
        return torch.from_numpy(out)


def _worker(rank, world, port, kind, out, reduce="data"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = O.ogrid(7, 5, 5, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0, 4.5, 6.0))
    consts = O.grav_constants() if kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    lo, hi = partition_layers(g.nz, world)[rank]
    op = ShardedOperator(OracleLocal(g, kind, consts, lo, hi), reduce=reduce)
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


@pytest.mark.parametrize("reduce", ["data", "spectrum"])
@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_two_rank_layer_sharding_matches_unsharded(kind, reduce):
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), kind, out, reduce), nprocs=world, join=True)
        d, xt = out["d"], out["xt"]
    g = O.ogrid(7, 5, 5, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0, 4.5, 6.0))
    consts = O.grav_constants() if kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    fw, tr = O.build_spectra(g, kind, consts)
    rng = np.random.default_rng(3)
    x = rng.uniform(size=g.n)
    v = rng.uniform(size=g.m)
    assert O.rel_l2(O.forward(g, fw, x), d) <= 1e-14
    if reduce == "data":
        assert np.array_equal(O.transpose(g, tr, v), xt)
    else:  # same per-layer arithmetic from the broadcast spectrum
        assert O.rel_l2(O.transpose(g, tr, v), xt) <= 1e-14


def _cgls_worker(rank, world, port, kind, damp, out):
    from paper_1912_06976_b200.parallel import sharded_cgls

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = O.ogrid(7, 5, 5, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0, 4.5, 6.0))
    consts = O.grav_constants() if kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    lo, hi = partition_layers(g.nz, world)[rank]
    op = ShardedOperator(OracleLocal(g, kind, consts, lo, hi))
    d = np.random.default_rng(21).normal(size=g.m)
    # only the root's data matters: the others' copies are overwritten by the broadcast
    dt = torch.from_numpy(d.copy()) if rank == 0 else torch.zeros(g.m, dtype=torch.float64)
    m_loc, hist = sharded_cgls(op, dt, iters=6, damp=damp)
    parts = [None] * world
    dist.all_gather_object(parts, m_loc.numpy())
    if rank == 0:
        out["m"] = np.concatenate(parts)
        out["hist"] = hist.numpy()[0]
    dist.destroy_process_group()


@pytest.mark.parametrize("damp", [0.0, 0.3])
@pytest.mark.parametrize("kind", ["gravity", "magnetic"])
def test_two_rank_layer_sharded_cgls_matches_oracle(kind, damp):
    """Layer-sharded CGLS over 2 gloo ranks (BASELINE configs[4]) equals the
    oracle's single-process CGLS: models to 1e-12, residual history to 1e-12."""
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_cgls_worker, args=(world, _free_port(), kind, damp, out), nprocs=world, join=True)
        m, hist = out["m"], out["hist"]
    g = O.ogrid(7, 5, 5, 1, 2, 2, 0, 1.0, 1.5, (0.0, 1.0, 2.5, 4.0, 4.5, 6.0))
    consts = O.grav_constants() if kind == "gravity" else O.mag_constants(33.0, 47.0, 45000.0)
    fw, tr = O.build_spectra(g, kind, consts)
    d = np.random.default_rng(21).normal(size=g.m)
    m_ref, h_ref = O.cgls(g, fw, tr, d, 6, damp=damp)
    assert O.rel_l2(m_ref, m) <= 1e-12
    np.testing.assert_allclose(hist, h_ref, rtol=1e-12)
    if damp == 0.0:
        assert hist[-1] < hist[0]
