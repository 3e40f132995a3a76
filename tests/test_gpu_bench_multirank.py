"""The N > 1 bench path (torchrun, layer shards, exchange, pipelined e2e,
max over ranks) on a single-GPU box: both ranks pinned to cuda:0 with the
gloo backend (BTTB_BENCH_DEVICE / BTTB_BENCH_BACKEND test knobs; the ranks'
kernels never wait on one another).  Checks the contract keys of the line
rank 0 prints, for both exchanges and the reference arm."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(*extra):
    env = dict(os.environ, BTTB_BENCH_DEVICE="0", BTTB_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-variants", *extra]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("reduce", ["data", "spectrum"])
def test_two_rank_bench_line(reduce):
    d = _run("--reduce", reduce)
    assert d["n_gpus"] == 2 and d["config"]["layers_per_rank"] == 64
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 64 * 1000 * 1000 * 8 + 1000 * 1000 * 8
    assert ("spectra" in d["config"]["exchange"]) == (reduce == "spectrum")


def test_two_rank_reference_arm():
    d = _run("--impl", "reference")
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0


def test_two_rank_layer_sharded_cgls():
    """--cgls under torchrun shards the depth layers (BASELINE configs[4]):
    16 of C5's 32 layers per rank, all 64 models on every rank, and the
    residual still drops like the single-GPU loop's."""
    d = _run("--config", "C5", "--dtype", "f32", "--cgls", "3")
    assert d["n_gpus"] == 2 and d["config"]["layers_per_rank"] == 16 and d["config"]["models_per_rank"] == 64
    assert d["config"]["parallelism"].startswith("layer-shard x2")
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert 0 < d["residual_drop_median"] < 0.9
