"""Benchmark of the B200 fast BTTB operator: G*m + G^T*d voxels/s and % HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--dtype f64|f32]
    python bench.py --impl reference ...        # the reference's CPU path (oracle port)

One step = one forward G*m and one transpose G^T*d over the configured
workload (BASELINE.json config C4 by default: magnetic, 1000x1000 stations,
128 layers, 1999x1999 embedding at 2048x2048 FFT lengths).  Under torchrun every rank holds a
contiguous block of depth layers (strong scaling: the workload is fixed); the
forward partial station vectors are summed with one NCCL all-reduce and the
data vector is broadcast for the transpose (paper_1912_06976_b200/parallel.py).

Rank 0 prints one JSON line (the driver contract in the task statement).
Roofline: algorithmic bytes per application B = b*(n+m) + b*nz*mx*my
(SURVEY.md 8(d)), over the measured HBM copy peak in MEASURED_PEAKS.json.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "G·m + Gᵀ·d voxels/sec (fp64/fp32) at 1/2/4/8 B200; % HBM roofline"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-torch", action="store_true",
                    help="time e2e through the torch-level pipelined path (the N>1 path) on one GPU too")
    ap.add_argument("--reduce", default="data", choices=["data", "spectrum"],
                    help="N>1 forward/transpose exchange: all-reduce of station vectors (data) or of "
                         "the partial station half spectra + broadcast of the data spectrum (spectrum)")
    ap.add_argument("--graph", type=int, default=0, choices=[0, 1],
                    help="1: capture one step (the C-ABI launches on the plan's streams, joined by "
                         "events) in a CUDA graph and time its replays (single GPU)")
    ap.add_argument("--cgls", type=int, default=0, metavar="ITERS",
                    help="time the batched CGLS driver instead: one step = ITERS iterations (one "
                         "G*m and one G^T*d each) over the config's batch; under torchrun the depth "
                         "layers are sharded over the ranks (BASELINE configs[4]), one NCCL all-reduce "
                         "of the partial G*p plus the scalar reductions per iteration")
    ap.add_argument("--cgls-shard", default="layers", choices=["layers", "models"],
                    help="N>1 CGLS: shard depth layers (default) or models over replicated stacks")
    ap.add_argument("--profile-step", action="store_true",
                    help="after warm-up run ONE step between cudaProfilerStart/Stop and exit "
                         "(for ncu --profile-from-start off); prints nothing")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_dist(world, local):
    """One process per GPU over NCCL.  Test knobs (not for measurements):
    BTTB_BENCH_DEVICE pins every rank to one device and BTTB_BENCH_BACKEND=gloo
    swaps the backend, so the N > 1 host logic runs on a single-GPU box
    (ranks share the GPU, their kernels never wait on one another)."""
    import torch
    import torch.distributed as dist

    dev_env = os.environ.get("BTTB_BENCH_DEVICE")
    idx = int(dev_env) if dev_env is not None else local
    torch.cuda.set_device(idx)
    dev = torch.device("cuda", idx)
    if world > 1:
        backend = os.environ.get("BTTB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # communicator logging (ranks, channels, NVLS) goes to stderr, so a
            # scaling run can verify the communicator size; stdout stays one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def workload(cfg, O):
    sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, dz, kind, args, batch = O.CONFIGS[cfg]
    desc = (f"{cfg} {kind} stations {sx}x{sy}, volume {sx + pxl + pxr}x{sy + pyl + pyr}x{nz}, "
            f"d=({dx:g},{dy:g},{dz:g}) m" + (f", D={args[0]:g} I={args[1]:g} F={args[2]:g}" if args else "")
            + (f", batch {batch}" if batch > 1 else ""))
    return desc, batch


def csrc_digest():
    """sha256 (16 hex) of the CUDA sources: ties a committed ncu traffic figure to the kernels it measured."""
    import hashlib

    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_1912_06976_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def measured_traffic(cfg, dtype):
    """DRAM bytes per application from the committed ncu capture (profiles/traffic.json:
    dram__bytes_read.sum + dram__bytes_write.sum over one application's launches), or None
    when that capture was taken on different kernel sources than the ones running."""
    rec, src = profile_record(f"{cfg}_{dtype}")
    return (rec.get("bytes_per_apply") if rec else None), src


def profile_record(key):
    """A committed per-kernel ncu figure (profiles/traffic.json) for `key`, with
    its source; the figure is None when it was captured on other kernel sources."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            rec = json.load(fh).get(key)
    except (OSError, ValueError):
        return None, None
    if not isinstance(rec, dict):
        return None, None
    src = {"profile": rec.get("profile"), "csrc_sha": rec.get("csrc_sha"), "current_csrc_sha": csrc_digest()}
    if rec.get("csrc_sha") != src["current_csrc_sha"]:
        return None, dict(src, stale=True)
    return rec, src


def c5_cgls_variant(dev, steps):
    """BASELINE configs[4] on one GPU: 64 gravity models on 256x256x32, fp32,
    10 CGLS iterations (a G*m and a G^T*d each) in the device-resident loop
    (bttb_cgls), data = G of seeded N(0, 0.1) models.  The 64 models share
    each layer's spectrum, so per voxel the loop moves few bytes and the
    column FFTs bind: the roofline fraction is reported
    against HBM with the FP32-pipe fraction of the column kernels from the
    committed ncu capture beside it."""
    import torch

    import paper_1912_06976_b200 as B
    from oracle import bttb_oracle as O

    og = O.config_grid("C5")
    grid = B.make_grid(og.sx, og.sy, og.nz, 0, 0, 0, 0, og.dx, og.dy, og.z)
    batch, iters = O.CONFIGS["C5"][12], 10
    st = B.build_transform_stack(grid, B.KernelParams.gravity(), dtype="float32", device=dev.index)
    truth = torch.tensor(np.random.default_rng(1000).normal(0.0, 0.1, (batch, og.n)), dtype=torch.float32,
                         device=dev)
    d = B.apply(st, truth, "forward")
    for _ in range(3):
        B.cgls(st, d, iters=iters, history=False)
    torch.cuda.synchronize()
    reps = max(3, min(steps, 20))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        B.cgls(st, d, iters=iters, history=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    _, hist = B.cgls(st, d, iters=iters)
    st.close()
    peak, _ = peaks()
    napply = 2 * iters + 1
    rec, src = profile_record("C5_cgls_f32")
    return {"ms_per_loop": ms, "iterations": iters, "models": batch,
            "value": batch * og.n * iters / (ms * 1e-3), "unit": "voxels/s (per G*m + G^T*d pair)",
            "roofline_frac": napply * algorithmic_bytes(og, 4, batch) / (ms * 1e-3) / 1e9 / peak,
            "fp32_pipe_frac": rec.get("fp32_pipe_frac") if rec else None, "profile_source": src,
            "residual_drop_median": float(np.median(hist[:, -1] / hist[:, 0]))}


def algorithmic_bytes(g, b, batch):
    """B = b*batch*(n+m) + b*nz*mx*my per application."""
    return b * batch * (g.n + g.m) + b * g.nz * g.mx * g.my


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: an NVML thread reads them every ~5 ms (the timed region of a
    20-step C4 run is only ~70 ms, too short for nvidia-smi's 50 ms loop and
    its start-up); only samples after mark() -- the start of the timed
    region -- count.  Falls back to an nvidia-smi loop without NVML."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.thread = None
        self.samples = []
        self.t_mark = None
        self.max_mhz = None

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        props = torch.cuda.get_device_properties(self.index)
        bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        import threading

        try:
            nv, h = self._nvml_handle()
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception:
            self._start_smi()
            return
        self._stop = False

        def loop():
            while not self._stop:
                try:
                    mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((time.perf_counter(), mhz, [n for n, b in bits.items() if rs & b]))
                except Exception:
                    pass
                time.sleep(0.005)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def _start_smi(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def mark(self):
        """The timed region starts now."""
        self.t_mark = time.perf_counter()

    def stop(self):
        if self.thread is not None:
            self._stop = True
            self.thread.join(timeout=2)
            rows = [(m, r) for (tt, m, r) in self.samples if self.t_mark is None or tt >= self.t_mark]
            sm = [m for m, _ in rows]
            reasons = sorted({n for _, r in rows for n in r})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                    "samples": len(sm), "reasons": reasons, "source": "nvml, 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.count(",") >= 6]
        reasons = set()
        sm, mx = [], None
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons), "source": "nvidia-smi, 50 ms"}


# ---------------------------------------------------------------------------
# CPU arm: the reference algorithm (oracle port), threads over depth layers
# ---------------------------------------------------------------------------
def cpu_sample(cfg, steps, warmup, layers_hint=None):
    from concurrent.futures import ThreadPoolExecutor

    from oracle import bttb_oracle as O

    cores = os.cpu_count() or 1
    g_full = O.config_grid(cfg)
    kind, consts = O.config_kernel(cfg)
    nl = g_full.nz if layers_hint is None else min(g_full.nz, layers_hint)
    g = O.config_grid(cfg, nz=nl)
    x, d = O.make_inputs(cfg, g, batch=1)
    with ThreadPoolExecutor(cores) as pool:
        t0 = time.perf_counter()
        fw, tr = O.build_spectra_threaded(g, kind, consts, list(range(nl)), pool)
        t_build = time.perf_counter() - t0
        for _ in range(warmup):
            O.forward_threaded(g, fw, x[0], pool)
            O.transpose_threaded(g, tr, d[0], pool)
        tf = tt = 0.0
        for _ in range(steps):
            t0 = time.perf_counter()
            O.forward_threaded(g, fw, x[0], pool)
            t1 = time.perf_counter()
            O.transpose_threaded(g, tr, d[0], pool)
            tf += t1 - t0
            tt += time.perf_counter() - t1
    voxels = g.n  # one batch item of the sample
    return {"value": voxels * steps / (tf + tt), "unit": "voxels/s", "cores": cores,
            "sample": (f"{cfg} geometry with {nl} of {g_full.nz} layers, 1 model, numpy pocketfft "
                       f"(reference algorithm, oracle port), {cores} threads over layers; "
                       f"build {t_build:.2f}s, fwd {1e3 * tf / steps:.1f} ms, "
                       f"tra {1e3 * tt / steps:.1f} ms per step"),
            "fwd_s": tf / steps, "tra_s": tt / steps, "build_s": t_build}


def cpu_full(cfg, x, v, threads=None):
    """The reference algorithm (oracle port) over EVERY layer of the config on
    the given inputs: all spectra built, one forward and one transpose, layers
    threaded on the host cores with bounded memory (O.products_chunked).
    Returns (d, xt, info) with the per-phase seconds -- the bench's parity
    oracle and its full-configuration CPU baseline in one pass."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import bttb_oracle as O

    cores = threads or os.cpu_count() or 1
    g = O.config_grid(cfg)
    kind, consts = O.config_kernel(cfg)
    with ThreadPoolExecutor(cores) as pool:
        d, xt, tm = O.products_chunked(g, kind, consts, x, v, pool)
    tm["cores"] = cores
    return d, xt, tm


def run_reference(a):
    """The reference's CPU path on the FULL configuration (every layer of
    C4): the reference algorithm (pinned oracle port -- the reference is pure
    numpy) with its two complex128 spectrum stacks built once, then per step
    one forward and one transpose over all layers, layers threaded over the
    host cores.  The driver's K and W are honoured (capped at 30 steps and 5
    warm-up steps: each C4 step is ~7 s of 16-thread CPU work, so K=20, W=5
    is ~3 minutes)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import bttb_oracle as O

    desc, batch = workload(a.config, O)
    cores = os.cpu_count() or 1
    g = O.config_grid(a.config)
    kind, consts = O.config_kernel(a.config)
    x, d = O.make_inputs(a.config, g, batch=1)
    steps = max(1, min(a.steps, 30))
    warm = max(0, min(a.warmup, 5))
    with ThreadPoolExecutor(cores) as pool:
        t0 = time.perf_counter()
        fw, tr = O.build_spectra_threaded(g, kind, consts, list(range(g.nz)), pool)
        t_build = time.perf_counter() - t0
        for _ in range(warm):
            O.forward_threaded(g, fw, x[0], pool)
            O.transpose_threaded(g, tr, d[0], pool)
        tf = tt = 0.0
        for _ in range(steps):
            t0 = time.perf_counter()
            O.forward_threaded(g, fw, x[0], pool)
            t1 = time.perf_counter()
            O.transpose_threaded(g, tr, d[0], pool)
            tf += t1 - t0
            tt += time.perf_counter() - t1
    value = g.n * steps / (tf + tt)
    sample = (f"{a.config}: all {g.nz} layers, 1 model, both complex128 spectrum stacks resident "
              f"({2 * g.nz * g.mx * g.my * 16 / 1e9:.1f} GB), numpy pocketfft (reference algorithm, oracle "
              f"port), {cores} threads over layers; build {t_build:.1f} s, fwd {1e3 * tf / steps:.0f} ms, "
              f"tra {1e3 * tt / steps:.0f} ms per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxels/s",
        "n_gpus": a.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * (tf + tt) / steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded (SURVEY.md 8(d))",
        "config": {"workload": desc, "sample": sample, "same_config": True},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_1912_06976_b200 as B
    from oracle import bttb_oracle as O  # input recipe + cpu baseline only
    from paper_1912_06976_b200.parallel import DeviceOperator, ShardedOperator, partition_layers

    rank, world, local = dist_env()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    dev = init_dist(world, local)
    cfg = a.config
    desc, batch = workload(cfg, O)
    og = O.config_grid(cfg)
    kind, _ = O.config_kernel(cfg)
    sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, dz, _, kargs, _ = O.CONFIGS[cfg]
    grid = B.make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, og.z)
    params = B.KernelParams.gravity() if kind == "gravity" else B.KernelParams.magnetic(*kargs)
    lo, hi = partition_layers(nz, world)[rank]
    np_dt = np.float64 if a.dtype == "f64" else np.float32
    t_dt = torch.float64 if a.dtype == "f64" else torch.float32
    bsz = 8 if a.dtype == "f64" else 4

    def build(dtype):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = B.build_transform_stack(grid, params, dtype="float64" if dtype == "f64" else "float32",
                                     device=dev.index, layers=(lo, hi))
        torch.cuda.synchronize()
        return st, time.perf_counter() - t0

    stack, t_build = build(a.dtype)
    op = ShardedOperator(DeviceOperator(stack), reduce=a.reduce)
    n_r = grid.n_r
    # seeded inputs, generated on the host (the model slice of this rank), resident in HBM
    rng = np.random.default_rng(1000 + rank)
    if cfg in ("C4",):
        xh = rng.uniform(0.0, 0.05, (batch, (hi - lo) * n_r))
    elif cfg == "C5":
        xh = rng.normal(0.0, 0.1, (batch, (hi - lo) * n_r))
    else:
        xh = rng.uniform(0.0, 1.0, (batch, (hi - lo) * n_r))
    dh = np.random.default_rng(1).normal(0.0, 1.0, (batch, grid.m))
    x_pin = torch.from_numpy(xh.astype(np_dt)).pin_memory()
    d_pin = torch.from_numpy(dh.astype(np_dt)).pin_memory()
    x = x_pin.to(dev)
    d = d_pin.to(dev)
    y = torch.empty((batch, grid.m), dtype=t_dt, device=dev)
    xt = torch.empty((batch, (hi - lo) * n_r), dtype=t_dt, device=dev)
    dwork = torch.empty_like(d)
    xs = x if batch > 1 else x[0]
    ys = y if batch > 1 else y[0]
    ds = dwork if batch > 1 else dwork[0]
    xts = xt if batch > 1 else xt[0]

    def step():
        op.forward(xs, ys)
        ds.copy_(d if batch > 1 else d[0])
        op.transpose(ds, xts)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, a.warmup)):
        step()
    barrier()
    if a.profile_step:
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        if world > 1:
            dist.destroy_process_group()
        return
    run = step
    if a.graph and world == 1:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            step()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=cap):
                step()
        torch.cuda.synchronize()
        run = graph.replay
        for _ in range(3):
            run()
        barrier()
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.15)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    sampler.mark()
    e0.record(stream)
    for _ in range(a.steps):
        run()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / a.steps
    launches_per_apply = stack.info()[9]
    # per-mode times (after the timed region; same stream, CUDA events)
    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(reps):
            fn()
        s1.record(stream)
        s1.synchronize()
        return s0.elapsed_time(s1) / reps

    reps = max(3, min(a.steps, 20))
    fwd_ms = timed(lambda: DeviceOperator.forward(op.local, xs, ys), reps)
    launch_fwd = stack.info()[9]
    tra_ms = timed(lambda: DeviceOperator.transpose(op.local, ds, xts), reps)
    launch_tra = stack.info()[9]

    # end-to-end through the public C ABI with host (pinned) buffers
    e2e = None
    if not a.no_e2e:
        yo = torch.empty((batch, grid.m), dtype=t_dt).pin_memory()
        xo = torch.empty((batch, (hi - lo) * n_r), dtype=t_dt).pin_memory()
        from paper_1912_06976_b200.multiply import apply_into

        def e2e_step():
            apply_into(stack, "forward", x_pin.data_ptr(), yo.data_ptr(), batch, host=True)
            if world > 1:
                t = yo.to(dev)
                dist.all_reduce(t)
                yo.copy_(t)
            apply_into(stack, "transpose", d_pin.data_ptr(), xo.data_ptr(), batch, host=True)

        # single GPU: the asynchronous host path (BTTB_HOST_ASYNC) -- every step
        # still copies its inputs in and its results out, but one step's
        # device-to-host copy overlaps the next step's host-to-device copy
        e2e_async = world == 1
        cur = torch.cuda.current_stream().cuda_stream

        def e2e_step_async():
            apply_into(stack, "forward", x_pin.data_ptr(), yo.data_ptr(), batch, cur, host="async-unordered")
            apply_into(stack, "transpose", d_pin.data_ptr(), xo.data_ptr(), batch, cur, host="async-unordered")

        # several GPUs (or --e2e-torch): the same pipelining one level up --
        # pinned host tensors copied on a side stream into two alternating device
        # buffer sets, the sharded operator (NCCL exchange included) on the
        # compute stream, results copied out on a second side stream
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        sets = [dict(x=torch.empty_like(x), d=torch.empty_like(d), y=torch.empty_like(y),
                     xt=torch.empty_like(xt)) for _ in range(2)]
        done_in = [torch.cuda.Event(), torch.cuda.Event()]
        done_comp = [torch.cuda.Event(), torch.cuda.Event()]
        done_out = [torch.cuda.Event(), torch.cuda.Event()]
        slot = [0]
        comp = torch.cuda.current_stream()

        def e2e_step_torch():
            i = slot[0]
            slot[0] ^= 1
            b = sets[i]
            with torch.cuda.stream(s_in):
                s_in.wait_event(done_comp[i])  # the set's previous compute has read x / d
                b["x"].copy_(x_pin, non_blocking=True)
                b["d"].copy_(d_pin, non_blocking=True)
                done_in[i].record(s_in)
            comp.wait_event(done_in[i])
            comp.wait_event(done_out[i])  # the set's previous results have left
            xs_, ys_, ds_, xts_ = ((b["x"], b["y"], b["d"], b["xt"]) if batch > 1
                                   else (b["x"][0], b["y"][0], b["d"][0], b["xt"][0]))
            op.forward(xs_, ys_)
            op.transpose(ds_, xts_)
            done_comp[i].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done_comp[i])
                yo.copy_(b["y"], non_blocking=True)
                xo.copy_(b["xt"], non_blocking=True)
                done_out[i].record(s_out)

        if a.e2e_torch or world > 1:
            e2e_async = False
            run_e2e = e2e_step_torch
        else:
            run_e2e = e2e_step_async if e2e_async else e2e_step
        run_e2e()
        # the same K steps as the device-timed loop (capped): the region is bracketed by
        # synchronisation, so it includes the pipeline's fill (first input copy) and drain
        # (last output copy) -- ~19 ms at C4, amortised over the K steps
        e_steps = max(2, min(a.steps, 50))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            run_e2e()
        barrier()
        t_e2e = (time.perf_counter() - t0) / e_steps
        if world > 1:
            tt = torch.tensor([t_e2e], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": batch * grid.n / t_e2e, "unit": "voxels/s",
               "h2d_bytes_per_step": int(x_pin.numel() * bsz + d_pin.numel() * bsz),
               "d2h_bytes_per_step": int(yo.numel() * bsz + xo.numel() * bsz),
               "ms_per_step": 1e3 * t_e2e, "steps": e_steps,
               "path": ("C ABI host pointers, asynchronous (copies of consecutive calls overlap)" if e2e_async
                        else "pinned host tensors, side-stream copies into two alternating device buffer sets, "
                             "sharded operator (copies of consecutive steps overlap)")}
        if world == 1:
            # the unchanged reference call: apply(stack, numpy array, mode) per
            # product -- pageable host arrays in, a new numpy array out, synchronous
            # (each call's copies cross PCIe in one direction, so consecutive calls
            # cannot overlap the way the asynchronous path above does)
            x_np, d_np = x_pin.numpy()[0].copy(), d_pin.numpy()[0].copy()
            B.apply(stack, x_np, "forward")
            B.apply(stack, d_np, "transpose")
            n_ref = 3
            t0 = time.perf_counter()
            for _ in range(n_ref):
                B.apply(stack, x_np, "forward")
                B.apply(stack, d_np, "transpose")
            t_ref = (time.perf_counter() - t0) / n_ref
            e2e["reference_api"] = {
                "value": grid.n / t_ref, "ms_per_step": 1e3 * t_ref,
                "path": "apply(stack, numpy_array, mode) as the reference's callers make it: pageable numpy "
                        "arrays, synchronous host path (BTTB_HOST_PTR: pinned chunk ring, four layer ranges whose "
                        "copies and compute overlap), new output array per call"}

    # max over ranks
    vals = torch.tensor([ms, fwd_ms, tra_ms, t_build], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, fwd_ms, tra_ms, t_build = vals.tolist()

    variants = {}
    variant_out = {}
    if not a.no_variants and cfg == "C4":
        other = "f32" if a.dtype == "f64" else "f64"
        st2, tb2 = build(other)
        op2 = DeviceOperator(st2)
        o_dt = torch.float32 if other == "f32" else torch.float64
        x2, d2 = xs.to(o_dt), ds.to(o_dt)
        y2 = torch.empty_like(ys, dtype=o_dt)
        xt2 = torch.empty_like(xts, dtype=o_dt)

        def step2():
            op2.forward(x2, y2)
            if world > 1:
                dist.all_reduce(y2)
                dist.broadcast(d2, 0)
            op2.transpose(d2, xt2)

        for _ in range(3):
            step2()
        barrier()
        r2 = max(3, min(a.steps, 50))
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(r2):
            step2()
        s1.record(stream)
        barrier()
        ms2 = s0.elapsed_time(s1) / r2
        b2 = 8 if other == "f64" else 4
        peak, _ = peaks()
        variants[other] = {"ms_per_step": ms2, "value": batch * grid.n / (ms2 * 1e-3),
                           "roofline_frac": 2 * algorithmic_bytes(og, b2, batch) / (ms2 * 1e-3) / 1e9 / peak,
                           "build_s": tb2}
        variant_out[other] = (y2.reshape(-1, grid.m)[0].double().cpu().numpy(),
                              xt2.reshape(-1, xt2.shape[-1])[0].double().cpu().numpy())
        st2.close()

    if not a.no_variants and cfg == "C4" and world == 1:
        variants["C5_cgls_f32"] = c5_cgls_variant(dev, a.steps)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    B_apply = algorithmic_bytes(og, bsz, batch)
    achieved = 2 * B_apply / (ms * 1e-3) / 1e9
    traffic, traffic_src = measured_traffic(cfg, a.dtype)
    # second floor of the fp64 step: its FP64 thread instructions at the pipe's
    # peak issue rate (committed ncu capture of the same kernel sources)
    fp64_rec, _ = profile_record(f"{cfg}_{a.dtype}_fp64_pipe") if world == 1 else (None, None)
    fp64_floor = None
    if fp64_rec:
        fp64_floor = {"floor_ms_per_step": fp64_rec["floor_ms_per_step"],
                      "fp64_thread_inst_per_step": fp64_rec["fp64_thread_inst_per_step"],
                      "pipe_busy_frac": fp64_rec["floor_ms_per_step"] / ms,
                      "profile": fp64_rec.get("profile"),
                      "note": "DADD + DMUL + DFMA thread instructions of one step / (148 SMs x 64 lanes per cycle); "
                              "the HBM floor of the algorithmic bytes is %.2f ms" % (2 * B_apply / peak / 1e6)}
    cpu = None
    parity = None
    if not a.no_cpu_baseline and world == 1:
        if cfg in ("C4", "C5"):
            # the reference algorithm over EVERY layer on the bench's own inputs:
            # parity oracle of the benched step and full-configuration CPU baseline
            y_gpu = y[0].double().cpu().numpy()
            xt_gpu = xt[0].double().cpu().numpy()
            d_ref, xt_ref, tm = cpu_full(cfg, xh[0], dh[0])
            from oracle import bttb_oracle as O2
            gate = 1e-10 if a.dtype == "f64" else 1e-5
            parity = {"fwd_rel_l2": O2.rel_l2(d_ref, y_gpu), "tra_rel_l2": O2.rel_l2(xt_ref, xt_gpu),
                      "gate": gate,
                      "oracle": f"reference algorithm (oracle port) over all {nz} layers on the benched inputs "
                                f"(model seed 1000, data seed 1), fp64"}
            parity["pass"] = bool(parity["fwd_rel_l2"] <= gate and parity["tra_rel_l2"] <= gate)
            for name, (yv, xv) in variant_out.items():
                g2 = 1e-10 if name == "f64" else 1e-5
                variants[name]["parity"] = {"fwd_rel_l2": O2.rel_l2(d_ref, yv), "tra_rel_l2": O2.rel_l2(xt_ref, xv),
                                            "gate": g2}
            cpu = {"value": grid.n / (tm["fwd_s"] + tm["tra_s"]), "unit": "voxels/s", "cores": tm["cores"],
                   "kind": "port",
                   "sample": (f"{cfg}: all {nz} layers (the full benched configuration, not extrapolated), "
                              f"1 model, numpy pocketfft (reference algorithm, oracle port), {tm['cores']} "
                              f"threads over layers, spectra built chunk by chunk; build {tm['build_s']:.1f} s, "
                              f"fwd {1e3 * tm['fwd_s']:.0f} ms, tra {1e3 * tm['tra_s']:.0f} ms")}
        else:
            cpu = cpu_sample(cfg, 1, 1, None)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "sample")} | {"kind": "port"}
    line = {
        "metric": METRIC,
        "value": batch * grid.n / (ms * 1e-3),
        "unit": "voxels/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": max(3, a.warmup),
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": a.dtype,
        "data": "synthetic, seeded host-generated inputs resident in HBM (no dataset exists; SURVEY.md 8(d))",
        "config": {"workload": desc, "fft_shape": list(stack.fft_shape),
                   "layers_per_rank": hi - lo, "parallelism": f"layer-shard x{world}",
                   "exchange": "none" if world == 1 else (
                       "all-reduce of partial station vectors + broadcast of the data vector" if a.reduce == "data"
                       else "all-reduce of partial station half spectra + broadcast of the data half spectrum"),
                   "l2": "inputs larger than L2 (spectra %.2f GB + model %.2f GB per rank)" % (
                       stack.device_bytes / 1e9,
                       x.numel() * bsz / 1e9),
                   "step": "1 forward (+all-reduce) + 1 transpose (+broadcast)"
                           + (", CUDA-graph replay" if (a.graph and world == 1) else "")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "frac_of_8TBs_nameplate": achieved / 8000.0,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_apply": B_apply, "fp64_pipe": fp64_floor,
                     "kernel": "operator step (row R2C -> column FFT*S accumulate -> column IFFT -> row C2R; both "
                               "directions), dominant kernels k_col_fwd_tma / k_col_tra_tma"},
        "fwd_ms": fwd_ms, "tra_ms": tra_ms, "build_s": t_build,
        "fwd_voxels_per_s": batch * grid.n / (fwd_ms * 1e-3),
        "tra_voxels_per_s": batch * grid.n / (tra_ms * 1e-3),
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": int((launch_fwd + launch_tra) * a.steps),
        "launches_per_step": int(launch_fwd + launch_tra),
        "variants": variants,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CGLS arm (--cgls ITERS): SURVEY.md 8(f)3, BASELINE config C5
# ---------------------------------------------------------------------------
def cgls_cpu_sample(cfg, iters):
    """The oracle's CGLS (numpy, 1 thread) on ONE model of the config's geometry."""
    from oracle import bttb_oracle as O

    g = O.config_grid(cfg)
    kind, consts = O.config_kernel(cfg)
    fw, tr = O.build_spectra(g, kind, consts)
    d = np.random.default_rng(1).normal(0.0, 1.0, g.m)
    it = max(1, min(iters, 3))
    t0 = time.perf_counter()
    O.cgls(g, fw, tr, d, it)
    dt = time.perf_counter() - t0
    return {"value": g.n * it / dt, "unit": "voxels/s", "cores": 1, "kind": "port",
            "sample": f"{cfg} geometry, 1 model, {it} CGLS iterations of the oracle (numpy pocketfft, "
                      f"reference algorithm per product), {dt:.2f} s"}


def run_cgls(a):
    import torch
    import torch.distributed as dist

    import paper_1912_06976_b200 as B
    from oracle import bttb_oracle as O  # input recipe + cpu baseline only

    rank, world, local = dist_env()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    dev = init_dist(world, local)
    cfg, iters = a.config, a.cgls
    desc, batch = workload(cfg, O)
    og = O.config_grid(cfg)
    kind, _ = O.config_kernel(cfg)
    sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, dz, _, kargs, _ = O.CONFIGS[cfg]
    grid = B.make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, og.z)
    params = B.KernelParams.gravity() if kind == "gravity" else B.KernelParams.magnetic(*kargs)
    np_dt = np.float64 if a.dtype == "f64" else np.float32
    bsz = 8 if a.dtype == "f64" else 4
    sdt = "float64" if a.dtype == "f64" else "float32"
    layer_shard = world > 1 and a.cgls_shard == "layers"
    if layer_shard:
        # BASELINE configs[4]: depth layers sharded, every rank iterates all models
        from paper_1912_06976_b200.parallel import DeviceOperator, ShardedOperator, partition_layers, sharded_cgls

        lo, hi = partition_layers(nz, world)[rank]
        b0, b1 = 0, batch
    else:
        # one GPU, or models sharded over ranks (replicas of the whole stack)
        lo, hi = 0, nz
        b0, b1 = batch * rank // world, batch * (rank + 1) // world
    nb = b1 - b0
    t0 = time.perf_counter()
    stack = B.build_transform_stack(grid, params, dtype=sdt, device=dev.index, layers=(lo, hi))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    # data of the batch: G applied to seeded N(0, 0.1) models (the C5 recipe) plus noise
    rng = np.random.default_rng(1000)
    truth = rng.normal(0.0, 0.1, (batch, grid.n))[b0:b1, lo * grid.n_r:hi * grid.n_r]
    tdt = torch.float64 if a.dtype == "f64" else torch.float32
    if layer_shard:
        sop = ShardedOperator(DeviceOperator(stack))
        dgen = sop.forward(torch.tensor(truth, device=dev, dtype=tdt).contiguous())
    else:
        dgen = B.apply(stack, torch.tensor(truth, device=dev), "forward")
    dgen += 1e-3 * dgen.abs().max() * torch.randn(dgen.shape, generator=torch.Generator(device=dev).manual_seed(7),
                                                   device=dev, dtype=dgen.dtype)
    d_dev = dgen.contiguous()
    d_pin = d_dev.cpu().pin_memory()

    if layer_shard:
        def step():
            return sharded_cgls(sop, d_dev, iters=iters, history=False)[0]
    else:
        def step():
            return B.cgls(stack, d_dev, iters=iters, history=False)[0]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, a.warmup)):
        step()
    barrier()
    if a.profile_step:
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        if world > 1:
            dist.destroy_process_group()
        return
    run = step
    if a.graph and not layer_shard:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            step()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=cap):
                step()
        torch.cuda.synchronize()
        run = graph.replay
        for _ in range(3):
            run()
        barrier()
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.15)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    sampler.mark()
    e0.record(stream)
    for _ in range(a.steps):
        run()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / a.steps
    # one product of each kind for the launch count and the roofline split
    m_dev = step()
    d_host = d_pin.numpy()
    m_pin = torch.empty((nb, stack.n_local), dtype=d_pin.dtype).pin_memory()
    e_steps = max(2, min(a.steps, 5))
    if layer_shard:
        _, hist = sharded_cgls(sop, d_dev, iters=iters)
        hist = hist.cpu().numpy()
        launches = None  # per-product launches vary by plan; counted per product below

        def e2e_step():
            dd = d_pin.to(dev, non_blocking=True)
            m_pin.copy_(sharded_cgls(sop, dd, iters=iters, history=False)[0], non_blocking=True)
            torch.cuda.current_stream().synchronize()
    else:
        _, hist = B.cgls(stack, d_dev, iters=iters)
        launches = int(stack.info()[9])
        # end to end: pinned host data in, pinned host models out, through the C ABI host path
        from paper_1912_06976_b200.inversion import cgls_into

        def e2e_step():
            cgls_into(stack, d_pin.data_ptr(), m_pin.data_ptr(), nb, iters, host=True)
    e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e_steps):
        e2e_step()
    barrier()
    t_e2e = (time.perf_counter() - t0) / e_steps
    if launches is None:  # library kernels of one sharded loop: iters forward + iters+1 transpose products
        B.apply(stack, m_dev, "forward")
        lf = int(stack.info()[9])
        B.apply(stack, d_dev, "transpose")
        launches = lf * iters + int(stack.info()[9]) * (iters + 1)
    vals = torch.tensor([ms, t_e2e], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, t_e2e = vals.tolist()
    if rank != 0:
        dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    B_apply = algorithmic_bytes(og, bsz, batch)
    # per iteration: one forward + one transpose (+ one transpose to start)
    napply = 2 * iters + 1
    achieved = napply * B_apply / (ms * 1e-3) / 1e9
    cpu = None if (a.no_cpu_baseline or world > 1) else cgls_cpu_sample(cfg, iters)
    rel_drop = float(np.median(hist[:, -1] / hist[:, 0]))
    line = {
        "metric": METRIC, "value": batch * grid.n * iters / (ms * 1e-3), "unit": "voxels/s",
        "n_gpus": world, "steps": a.steps, "warmup": max(3, a.warmup), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
        "data": "synthetic: seeded N(0,0.1) models through the operator plus 0.1% noise, resident in HBM",
        "config": {"workload": desc, "step": f"{iters} CGLS iterations (G*m + G^T*d each) over the batch"
                   + (", CUDA-graph replay" if a.graph else ""),
                   "fft_shape": list(stack.fft_shape), "models_per_rank": nb, "layers_per_rank": hi - lo,
                   "parallelism": (f"layer-shard x{world} (NCCL all-reduce of G*p + scalars per iteration)"
                                   if layer_shard else f"model-shard x{world} (replicated stack)"
                                   if world > 1 else "single GPU, device-resident loop (bttb_cgls)"),
                   "l2": "per-iteration vectors (%.2f GB) larger than L2" % (3 * nb * grid.n * bsz / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind, "traffic": None,
                     "algorithmic_bytes_per_apply": B_apply,
                     "kernel": "CGLS loop: fused operator products + fused vector updates"},
        "build_s": t_build, "residual_drop_median": rel_drop,
        "cpu_baseline": cpu,
        "e2e": {"value": batch * grid.n * iters / t_e2e, "unit": "voxels/s",
                "h2d_bytes_per_step": int(d_host.size * bsz), "d2h_bytes_per_step": int(nb * stack.n_local * bsz),
                "ms_per_step": 1e3 * t_e2e},
        "clocks": clocks,
        "gpu_launches": launches * a.steps, "launches_per_step": launches,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.cgls > 0:
        run_cgls(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
