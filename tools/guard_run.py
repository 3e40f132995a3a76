"""Guard-zone / boundary sweep of the operator (run by tests/test_gpu_guards.py).

Runs with BTTB_GUARD=1 (64 KB pattern zones around every plan buffer and the
spectrum cache, checked by bttb_debug_check_guards) over every plan family --
the reference's padded 6x5x2 grids, C1, C2, C3, a C4 layer block at 2048^2
and at 2000^2, C5 batched fp32 -- in both dtypes, through every entry: numpy
host path, device tensors written into the middle of NaN-filled arenas (a
write outside the output range shows up as a changed canary), the staged
split products, both asynchronous host modes and CGLS.  Each case is also
checked against the oracle at the parity gate.  Prints one line per case and
exits non-zero on the first failure.  Stand-in for compute-sanitizer memcheck,
which this GPU pool does not allow.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BTTB_GUARD", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_06976_b200 as B  # noqa: E402
from paper_1912_06976_b200 import _lib  # noqa: E402
from paper_1912_06976_b200.multiply import apply_into  # noqa: E402
from paper_1912_06976_b200.parallel import DeviceOperator  # noqa: E402
from oracle import bttb_oracle as O  # noqa: E402

CANARY = 1 << 14  # elements of NaN canary on each side of a device output
TOL = {"float64": 1e-10, "float32": 1e-5}


def guards(st):
    bad = _lib.lib().bttb_debug_check_guards(st.handle)
    if bad != 0:
        raise SystemExit(f"guard zones overwritten in {bad} plan buffers")


def arena(n, tdt):
    a = torch.full((n + 2 * CANARY,), float("nan"), dtype=tdt, device="cuda")
    return a, a[CANARY:CANARY + n]


def canary_ok(a, n):
    return bool(torch.isnan(a[:CANARY]).all()) and bool(torch.isnan(a[CANARY + n:]).all())


def case(label, og, params, kind, consts, dtype, layers=None, shape=None, batch=1):
    lo, hi = layers or (0, og.nz)
    L = list(range(lo, hi))
    rng = np.random.default_rng(17)
    x = rng.uniform(0.0, 1.0, (batch, (hi - lo) * og.n_r))
    v = rng.normal(0.0, 1.0, (batch, og.m))
    q = lambda a: np.asarray(a, dtype=dtype).astype(np.float64)  # noqa: E731
    fw, tr = O.build_spectra(og, kind, consts, layers=L)
    want_f = np.stack([O.forward(og, fw, q(x[b]), layers=L) for b in range(batch)])
    want_t = np.stack([O.transpose(og, tr, q(v[b])) for b in range(batch)])
    grid = B.make_grid(og.sx, og.sy, og.nz, og.pxl, og.pxr, og.pyl, og.pyr, og.dx, og.dy, og.z)
    tdt = torch.float64 if dtype == "float64" else torch.float32
    tol = TOL[dtype] if kind == "gravity" or lo == 0 else max(TOL[dtype], 1e-8)
    with B.build_transform_stack(grid, params, dtype=dtype, layers=layers, fft_shape=shape) as st:
        guards(st)
        f = B.apply(st, x if batch > 1 else x[0], "forward")
        t = B.apply(st, v if batch > 1 else v[0], "transpose")
        guards(st)
        errs = [O.rel_l2(want_f.ravel(), np.ravel(f)), O.rel_l2(want_t.ravel(), np.ravel(t))]
        # device pointers into canary arenas
        nin, nout = batch * st.n_local, batch * og.m
        xa, xd = arena(nin, tdt)
        xd.copy_(torch.tensor(x.ravel(), dtype=tdt))
        ya, yd = arena(nout, tdt)
        s = torch.cuda.current_stream().cuda_stream
        apply_into(st, "forward", xd.data_ptr(), yd.data_ptr(), batch, s)
        va, vd = arena(nout, tdt)
        vd.copy_(torch.tensor(v.ravel(), dtype=tdt))
        ta, td = arena(nin, tdt)
        apply_into(st, "transpose", vd.data_ptr(), td.data_ptr(), batch, s)
        torch.cuda.synchronize()
        for a, n, what in ((ya, nout, "forward output"), (ta, nin, "transpose output"),
                           (xa, nin, "forward input"), (va, nout, "transpose input")):
            if not canary_ok(a, n):
                raise SystemExit(f"{label}: canary around the {what} overwritten")
        errs += [O.rel_l2(want_f.ravel(), yd.double().cpu().numpy()), O.rel_l2(want_t.ravel(), td.double().cpu().numpy())]
        # both asynchronous host modes
        for mode in ("async", "async-unordered"):
            xp = torch.tensor(x.ravel(), dtype=tdt).pin_memory()
            yp = torch.empty(nout, dtype=tdt).pin_memory()
            apply_into(st, "forward", xp.data_ptr(), yp.data_ptr(), batch, s, host=mode)
            torch.cuda.synchronize()
            errs.append(O.rel_l2(want_f.ravel(), yp.double().numpy()))
        guards(st)
        # staged split products (the multi-GPU exchange path)
        op = DeviceOperator(st)
        xs = torch.tensor(x if batch > 1 else x[0], dtype=tdt, device="cuda")
        vs = torch.tensor(v if batch > 1 else v[0], dtype=tdt, device="cuda")
        try:
            errs.append(O.rel_l2(want_f.ravel(),
                                 op.from_spectrum(op.forward_spectrum(xs)).double().cpu().numpy().ravel()))
            errs.append(O.rel_l2(want_t.ravel(),
                                 op.transpose_from_spectrum(op.transpose_spectrum(vs)).double().cpu().numpy().ravel()))
        except ValueError as exc:  # the generic-length path has no split products
            if "split products" not in str(exc):
                raise
        guards(st)
        if lo == 0 and hi == og.nz:
            B.cgls(st, v if batch > 1 else v[0], iters=2)
            guards(st)
    worst = max(errs)
    print(f"{label} {dtype}: worst rel-L2 {worst:.2e} over {len(errs)} products, guards and canaries intact",
          flush=True)
    if not worst <= tol:
        raise SystemExit(f"{label} {dtype}: parity {worst:.3e} > {tol}")


def main():
    only = sys.argv[1:]
    grav, gk = B.KernelParams.gravity(), ("gravity", O.grav_constants())
    mag = B.KernelParams.magnetic(33.0, 47.0, 45000.0)
    mk = ("magnetic", O.mag_constants(33.0, 47.0, 45000.0))
    cases = []
    for pads in [(0, 0, 0, 0), (2, 1, 1, 2), (3, 0, 0, 2)]:
        og = O.ogrid(6, 5, 2, *pads, 1.0, 1.5, (0.0, 1.0, 2.5))
        cases.append((f"small{pads}-grav", og, grav, *gk, {}))
        cases.append((f"small{pads}-mag", og, mag, *mk, {}))
    for name in ("C1", "C2", "C3"):
        kind, consts = O.config_kernel(name)
        p = grav if kind == "gravity" else B.KernelParams.magnetic(*O.CONFIGS[name][11])
        cases.append((name, O.config_grid(name), p, kind, consts, {}))
    c4 = O.config_grid("C4")
    k4, c4c = O.config_kernel("C4")
    p4 = B.KernelParams.magnetic(*O.CONFIGS["C4"][11])
    cases.append(("C4[0:2]", c4, p4, k4, c4c, {"layers": (0, 2)}))
    cases.append(("C4[126:128]-L2000", c4, p4, k4, c4c, {"layers": (126, 128), "shape": (2000, 2000)}))
    c5 = O.config_grid("C5", nz=4)
    cases.append(("C5x3", c5, grav, *gk, {"batch": 3}))
    for label, og, p, kind, consts, kw in cases:
        if only and not any(label.startswith(o) for o in only):
            continue
        for dtype in ("float64", "float32"):
            case(label, og, p, kind, consts, dtype, **kw)
    print("guard sweep clean", flush=True)


if __name__ == "__main__":
    main()
