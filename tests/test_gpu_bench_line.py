"""The default (N = 1) bench line: contract keys, the roofline object (live
achieved figure, traffic and FP64-pipe floor tagged with the profile they
came from) and the end-to-end leg -- on the headline configuration with a
few steps and without the CPU arm (tests/test_gpu_headline.py checks that
configuration against the oracle)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_single_gpu_bench_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--no-variants"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["metric"] and d["unit"] == "voxels/s" and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert "C4" in d["config"]["workload"] and d["config"]["fft_shape"] == [2048, 2048]
    n = 1000 * 1000 * 128
    assert abs(d["value"] - n / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert abs(r["achieved"] - 2 * r["algorithmic_bytes_per_apply"] / (d["ms_per_step"] * 1e-3) / 1e9) < 1e-6 * r["achieved"]
    src = r["traffic_source"]
    if src.get("stale"):
        assert r["traffic"] is None and r["fp64_pipe"] is None  # figures of other kernel sources are not reported
    else:
        assert r["traffic"] >= r["algorithmic_bytes_per_apply"]
        assert 0 < r["fp64_pipe"]["pipe_busy_frac"] < 1 and r["fp64_pipe"]["profile"] == src["profile"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == (n + 1000 * 1000) * 8 == e["d2h_bytes_per_step"]
    assert e["value"] < d["value"]  # the copies are inside the timed region
    assert d["gpu_launches"] == 3 * d["launches_per_step"] and d["launches_per_step"] >= 6
    assert d["clocks"]["sm_mhz"] > 0 and isinstance(d["clocks"]["reasons"], list)
