"""numpy restatement of the reference ``bttb`` hot path (arXiv 1912.06976).

TEST INFRASTRUCTURE ONLY -- the checker for the sm_100a product path and the
CPU arm of ``bench.py``.  Nothing in ``paper_1912_06976_b200`` imports it.

Citations are to ``/root/reference/pkg/src/bttb/*.py`` (file:line).  Every
floating-point expression keeps the reference's operation order so that the
restatement is bit-identical to the reference on the same numpy build; that is
pinned by ``tests/test_oracle_golden.py`` against vectors produced by the
reference itself (``tests/golden/make_golden.py``).

Layout conventions (``multiply.py:25-26``): model vectors are layer-major and
x-fastest (prism (p, q) of layer r at ``r*n_r + q*nx + p``); data vectors are
x-fastest (station (i, j) at ``j*sx + i``).
"""
from dataclasses import dataclass

import numpy as np

__all__ = [
    "GAMMA", "OGrid", "ogrid", "corner_vectors", "grav_constants",
    "mag_constants", "gravity_corner_sum", "magnetic_entries",
    "layer_window", "embed_window", "transpose_defining_array",
    "build_spectra", "forward", "transpose", "rel_l2", "make_inputs",
    "blob_model", "CONFIGS", "config_grid", "config_kernel", "cgls",
    "products_chunked", "layer_window_extended",
]

#: CODATA gravitational constant (``kernels.py:16``).
GAMMA = 6.67430e-11


# --------------------------------------------------------------------------
# geometry (grid.py:26-199)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class OGrid:
    """Geometry record; derived sizes follow ``grid.py:78-104``."""
    sx: int
    sy: int
    nz: int
    pxl: int
    pxr: int
    pyl: int
    pyr: int
    dx: float
    dy: float
    z: tuple

    @property
    def nx(self):
        return self.sx + self.pxl + self.pxr

    @property
    def ny(self):
        return self.sy + self.pyl + self.pyr

    @property
    def m(self):
        return self.sx * self.sy

    @property
    def n_r(self):
        return self.nx * self.ny

    @property
    def n(self):
        return self.n_r * self.nz

    @property
    def mx(self):
        return self.sx + self.nx - 1

    @property
    def my(self):
        return self.sy + self.ny - 1


def ogrid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, z):
    return OGrid(int(sx), int(sy), int(nz), int(pxl), int(pxr), int(pyl),
                 int(pyr), float(dx), float(dy), tuple(float(v) for v in z))


def corner_vectors(g, flavor):
    """Staggered corner distances.

    ``sym``  (grid.py:177-187): (l - 1/2)*d, l = 0 .. s+max(pad)   (inclusive)
    ``full`` (grid.py:190-199): (l - h + 1/2)*d, l = 0 .. 2h-1, h = s+max(pad)
    Entries are exact odd multiples of d/2 before the multiply by d.
    """
    hx = g.sx + max(g.pxl, g.pxr)
    hy = g.sy + max(g.pyl, g.pyr)
    if flavor == "sym":
        cx = (np.arange(hx + 1) - 0.5) * g.dx
        cy = (np.arange(hy + 1) - 0.5) * g.dy
    elif flavor == "full":
        cx = (np.arange(2 * hx) - hx + 0.5) * g.dx
        cy = (np.arange(2 * hy) - hy + 0.5) * g.dy
    else:
        raise ValueError(flavor)
    return cx, cy


def grav_constants(gamma=GAMMA, scale=1.0):
    """The single multiplier of ``kernels.py:98``: gamma*scale."""
    return gamma * scale


def mag_constants(D, I, F):
    """Five total-field constants, ``kernels.py:48-64``.

    x North, y East, z down; induced magnetization only.
    """
    Dr, Ir = np.radians(D), np.radians(I)
    cl = np.cos(Ir) * np.cos(Dr)
    cm = np.cos(Ir) * np.sin(Dr)
    cn = np.sin(Ir)
    ht = F / (4.0 * np.pi)
    return ht * np.array([2 * cm * cn, 2 * cl * cn, 2 * cl * cm,
                          cn * cn - cm * cm, cn * cn - cl * cl])


# --------------------------------------------------------------------------
# kernel-entry generation (kernels.py:81-155)
# --------------------------------------------------------------------------
def gravity_corner_sum(z1, z2, cx, cy, gs):
    """Vertical-gravity entries over a corner grid (``kernels.py:81-102``).

    Corner term CM = (CM56 - CMY - CMX)*gs with CMX = ln((x+R1)/(x+R2))*y,
    CMY = ln((y+R1)/(y+R2))*x, CM56 = atan2(xy, R1 z1) z1 - atan2(xy, R2 z2) z2;
    entry (p, q) = -(CM[p,q] - CM[p,q+1] - CM[p+1,q] + CM[p+1,q+1]).
    """
    X = cx[:, None]
    Y = cy[None, :]
    sq = X ** 2 + Y ** 2          # grid.py:173 (r2 table)
    prod = X * Y                  # grid.py:172 (xy table)
    R1 = np.sqrt(sq + z1 * z1)
    R2 = np.sqrt(sq + z2 * z2)
    tx = np.log((X + R1) / (X + R2)) * Y
    ty = np.log((Y + R1) / (Y + R2)) * X
    t56 = np.arctan2(prod, R1 * z1) * z1 - np.arctan2(prod, R2 * z2) * z2
    C = (t56 - ty - tx) * gs
    return -(C[:-1, :-1] - C[:-1, 1:] - C[1:, :-1] + C[1:, 1:])


def magnetic_entries(z1, z2, cx, cy, gc):
    """Total-field entries over a corner grid (``kernels.py:105-155``).

    Logs are taken of corner-product ratios grouped by corner parity
    (``kernels.py:121-135``); F4/F5 are signed sums of corner atan2 terms
    (``kernels.py:137-150``).  Operation order is the reference's.
    """
    sq = cx[:, None] ** 2 + cy[None, :] ** 2
    P1 = np.sqrt(sq + z1 * z1)
    P2 = np.sqrt(sq + z2 * z2)
    xa, xb = cx[:-1, None], cx[1:, None]
    ya, yb = cy[None, :-1], cy[None, 1:]

    def ratio(ta, tb, tc, td, sa, sb, sc, sd):
        # (even2 * odd1) / (even1 * odd2); even = corners (a,a),(b,b); odd = (b,a),(a,b)
        ev1 = (P1[:-1, :-1] + ta) * (P1[1:, 1:] + tb)
        od1 = (P1[1:, :-1] + tc) * (P1[:-1, 1:] + td)
        ev2 = (P2[:-1, :-1] + sa) * (P2[1:, 1:] + sb)
        od2 = (P2[1:, :-1] + sc) * (P2[:-1, 1:] + sd)
        return (ev2 * od1) / (ev1 * od2)

    f1 = ratio(xa, xb, xb, xa, xa, xb, xb, xa)
    f2 = ratio(ya, yb, ya, yb, ya, yb, ya, yb)
    f3 = ratio(z1, z1, z1, z1, z2, z2, z2, z2)

    def axz(P, z):
        return (np.arctan2(xb * z, P[1:, 1:] * yb)
                - np.arctan2(xa * z, P[:-1, 1:] * yb)
                - np.arctan2(xb * z, P[1:, :-1] * ya)
                + np.arctan2(xa * z, P[:-1, :-1] * ya))

    def ayz(P, z):
        return (np.arctan2(yb * z, P[1:, 1:] * xb)
                - np.arctan2(yb * z, P[:-1, 1:] * xa)
                - np.arctan2(ya * z, P[1:, :-1] * xb)
                + np.arctan2(ya * z, P[:-1, :-1] * xa))

    f4 = axz(P2, z2) - axz(P1, z1)
    f5 = ayz(P2, z2) - ayz(P1, z1)
    return (gc[0] * np.log(f1) + gc[1] * np.log(f2) + gc[2] * np.log(f3)
            + gc[3] * f4 + gc[4] * f5)


def layer_window(g, kind, consts, layer):
    """Response at every signed offset a layer needs (``kernels.py:158-184``).

    Window entry (a, b) is offset (a-(sx+pxl-1), b-(sy+pyl-1)).  Gravity is
    evaluated on the non-negative quadrant and mirrored by |offset|;
    magnetic is evaluated on the full corner slice.
    """
    z1, z2 = g.z[layer], g.z[layer + 1]
    if kind == "gravity":
        cx, cy = corner_vectors(g, "sym")
        q = gravity_corner_sum(z1, z2, cx, cy, consts)
        ax = np.abs(np.arange(g.mx) - (g.sx + g.pxl - 1))
        ay = np.abs(np.arange(g.my) - (g.sy + g.pyl - 1))
        return q[np.ix_(ax, ay)]
    cx, cy = corner_vectors(g, "full")
    hx = g.sx + max(g.pxl, g.pxr)
    hy = g.sy + max(g.pyl, g.pyr)
    sx_ = slice(hx - g.sx - g.pxl, hx + g.sx + g.pxr)
    sy_ = slice(hy - g.sy - g.pyl, hy + g.sy + g.pyr)
    return magnetic_entries(z1, z2, cx[sx_], cy[sy_], consts)


# --------------------------------------------------------------------------
# circulant embedding + spectra (transform.py:75-104)
# --------------------------------------------------------------------------
def embed_window(w, g):
    """T^circ: flip then cyclic shift by the station counts (``transform.py:85-88``)."""
    return np.roll(w[::-1, ::-1], (g.sx, g.sy), axis=(0, 1))


def transpose_defining_array(T):
    """T~[t] = T[-t] (``transform.py:75-82``)."""
    return np.roll(np.asarray(T)[::-1, ::-1], (1, 1), axis=(0, 1))


def build_spectra(g, kind, consts, layers=None):
    """Per-layer fft2 of T^circ and of its transpose layout (``transform.py:91-104``).

    ``layers`` selects a subset (for bounded samples of large configs).
    Returns (forward_list, transpose_list) of complex128 (mx, my) arrays.
    """
    idx = range(g.nz) if layers is None else layers
    fw, tr = [], []
    for r in idx:
        T = embed_window(layer_window(g, kind, consts, r), g)
        fw.append(np.fft.fft2(T))
        tr.append(np.fft.fft2(transpose_defining_array(T)))
    return fw, tr


# --------------------------------------------------------------------------
# products (multiply.py:22-57)
# --------------------------------------------------------------------------
def forward(g, fw, x, layers=None):
    """d = sum_r real(ifft2(That_r * fft2(embed(x_r))))[:sx, :sy] (``multiply.py:37-46``).

    ``layers`` lists the global layer index of each entry of ``fw``; ``x`` then
    holds exactly those layers' prisms (layer-major).
    """
    x = np.asarray(x, dtype=float)
    idx = list(range(g.nz)) if layers is None else list(layers)
    buf = np.zeros((g.mx, g.my))
    d = np.zeros(g.m)
    for k, _ in enumerate(idx):
        buf[:g.nx, :g.ny] = x[k * g.n_r:(k + 1) * g.n_r].reshape(g.ny, g.nx).T
        y = np.fft.ifft2(fw[k] * np.fft.fft2(buf))
        d += y.real[:g.sx, :g.sy].T.ravel()
    return d


def transpose(g, tr, v):
    """x_r = real(ifft2(That~_r * fft2(embed(v))))[:nx, :ny] (``multiply.py:47-57``)."""
    v = np.asarray(v, dtype=float)
    buf = np.zeros((g.mx, g.my))
    buf[:g.sx, :g.sy] = v.reshape(g.sy, g.sx).T
    vh = np.fft.fft2(buf)
    out = np.empty(len(tr) * g.n_r)
    for k, T in enumerate(tr):
        y = np.fft.ifft2(T * vh)
        out[k * g.n_r:(k + 1) * g.n_r] = y.real[:g.nx, :g.ny].T.ravel()
    return out


def rel_l2(a, b):
    """||a-b||/||a||; 0 if both zero, inf if only a is zero (``multiply.py:61-71``)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    na = np.linalg.norm(a)
    nd = np.linalg.norm(a - b)
    if na == 0.0:
        return 0.0 if nd == 0.0 else np.inf
    return nd / na


def cgls(g, fw, tr, d, iters, damp=0.0, rtol=1e-13):
    """Textbook CGLS on min |G m - d|^2 + damp^2 |m|^2 from m = 0 (the checker
    of ``bttb_cgls``; the reference has no inversion loop -- PAPER.md:640 names
    it future work, SPEC.md:320 a non-goal -- so this restates the standard
    algorithm over the pinned ``forward``/``transpose`` above).  Like the
    device loop it freezes (alpha = beta = 0) once |s_k| <= rtol |s_0|: past
    convergence CG only amplifies rounding noise.  Returns
    (m, [|r_0|, ..., |r_iters|])."""
    d = np.asarray(d, dtype=float)
    m = np.zeros(len(tr) * g.n_r)
    r = d.copy()
    s = transpose(g, tr, r)
    p = s.copy()
    gamma = float(s @ s)
    floor = rtol * rtol * gamma
    hist = [float(np.linalg.norm(r))]
    for _ in range(iters):
        q = forward(g, fw, p)
        delta = float(q @ q) + damp * damp * float(p @ p)
        alpha = gamma / delta if (delta > 0 and gamma > floor) else 0.0
        m = m + alpha * p
        r = r - alpha * q
        s = transpose(g, tr, r) - damp * damp * m
        gnew = float(s @ s)
        beta = gnew / gamma if gamma > floor else 0.0
        gamma = gnew
        p = s + beta * p
        hist.append(float(np.linalg.norm(r)))
    return m, hist


# --------------------------------------------------------------------------
# BASELINE.json configs and seeded inputs
# --------------------------------------------------------------------------
CONFIGS = {
    # name: (sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, dz, kind, kernel-args, batch)
    "C1": (50, 40, 10, 0, 0, 0, 0, 50.0, 50.0, 50.0, "gravity", (), 1),
    "C2": (50, 40, 10, 0, 0, 0, 0, 50.0, 50.0, 50.0, "magnetic", (3.0, 50.0, 50000.0), 1),
    "C3": (200, 160, 20, 10, 10, 8, 8, 100.0, 100.0, 100.0, "gravity", (), 1),
    "C4": (1000, 1000, 128, 0, 0, 0, 0, 25.0, 25.0, 20.0, "magnetic", (10.0, 60.0, 50000.0), 1),
    "C5": (256, 256, 32, 0, 0, 0, 0, 50.0, 50.0, 50.0, "gravity", (), 64),
}


def config_grid(name, nz=None):
    sx, sy, nz0, pxl, pxr, pyl, pyr, dx, dy, dz, _, _, _ = CONFIGS[name]
    nz = nz0 if nz is None else nz
    return ogrid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, [r * dz for r in range(nz + 1)])


def config_kernel(name):
    """(kind, consts) for a config: gamma*scale for gravity, gc[5] for magnetic."""
    kind, args = CONFIGS[name][10], CONFIGS[name][11]
    if kind == "gravity":
        return kind, grav_constants()
    return kind, mag_constants(*args)


def blob_model(g, seed=0, nblobs=8):
    """C3 model: sum of 8 isotropic Gaussian blobs on a zero background.

    centre ~ U over the (x, y, z) index box, amplitude ~ U[-0.5, 0.5],
    sigma ~ U[3, 15] cells; drawn in that order per blob from default_rng(seed).
    """
    rng = np.random.default_rng(seed)
    p = np.arange(g.nx)[None, None, :]
    q = np.arange(g.ny)[None, :, None]
    r = np.arange(g.nz)[:, None, None]
    out = np.zeros((g.nz, g.ny, g.nx))
    for _ in range(nblobs):
        c = rng.uniform([0, 0, 0], [g.nx, g.ny, g.nz])
        a = rng.uniform(-0.5, 0.5)
        s = rng.uniform(3.0, 15.0)
        out += a * np.exp(-((p - c[0]) ** 2 + (q - c[1]) ** 2 + (r - c[2]) ** 2) / (2 * s * s))
    return out.ravel()


def make_inputs(name, g=None, seed_model=0, seed_data=1, batch=None):
    """Seeded model (batch, n) and data (batch, m) vectors for a config."""
    g = config_grid(name) if g is None else g
    b = CONFIGS[name][12] if batch is None else batch
    rm = np.random.default_rng(seed_model)
    rd = np.random.default_rng(seed_data)
    if name == "C1":
        x = rm.uniform(0.0, 1.0, (b, g.n))
    elif name == "C2":
        x = rm.uniform(0.0, 0.1, (b, g.n))
    elif name == "C3":
        x = np.stack([blob_model(g, seed_model + k) for k in range(b)])
    elif name == "C4":
        x = rm.uniform(0.0, 0.05, (b, g.n))
    elif name == "C5":
        x = rm.normal(0.0, 0.1, (b, g.n))
    else:
        raise KeyError(name)
    d = rd.normal(0.0, 1.0, (b, g.m))
    return x, d


# --------------------------------------------------------------------------
# threaded layer loop (bench.py CPU arm).  numpy's pocketfft releases the GIL,
# so layers run concurrently; per-layer results are combined in layer order,
# giving exactly the serial loop's numbers.
# --------------------------------------------------------------------------
def build_spectra_threaded(g, kind, consts, layers, pool):
    pairs = list(pool.map(lambda r: build_spectra(g, kind, consts, [r]), layers))
    return [p[0][0] for p in pairs], [p[1][0] for p in pairs]


def forward_threaded(g, fw, x, pool):
    parts = list(pool.map(
        lambda k: forward(g, [fw[k]], x[k * g.n_r:(k + 1) * g.n_r], layers=[k]), range(len(fw))))
    d = np.zeros(g.m)
    for p in parts:
        d += p
    return d


def transpose_threaded(g, tr, v, pool):
    parts = list(pool.map(lambda T: transpose(g, [T], v), tr))
    return np.concatenate(parts)


def products_chunked(g, kind, consts, x, v, pool, chunk=16):
    """G x and G^T v over ALL layers of a large grid with bounded memory.

    The reference builds both full spectrum stacks and then loops over layers
    (transform.py:91-104, multiply.py:37-57); this runs the same per-layer
    arithmetic chunk by chunk (at most ``chunk`` layers' spectra alive, both
    stacks) with the layers of a chunk threaded.  Per-layer results are
    identical to the serial loop; the forward partials are summed chunk by
    chunk (layer order kept within a chunk).  Returns (d, xt, timings) with
    the build / forward / transpose seconds.
    """
    import time

    x = np.asarray(x, dtype=float)
    v = np.asarray(v, dtype=float)
    d = np.zeros(g.m)
    xt = np.empty(g.n)
    tb = tf = tt = 0.0
    for lo in range(0, g.nz, chunk):
        idx = list(range(lo, min(g.nz, lo + chunk)))
        t0 = time.perf_counter()
        fw, tr = build_spectra_threaded(g, kind, consts, idx, pool)
        t1 = time.perf_counter()
        d += forward_threaded(g, fw, x[lo * g.n_r:(lo + len(idx)) * g.n_r], pool)
        t2 = time.perf_counter()
        xt[lo * g.n_r:(lo + len(idx)) * g.n_r] = transpose_threaded(g, tr, v, pool)
        t3 = time.perf_counter()
        tb, tf, tt = tb + t1 - t0, tf + t2 - t1, tt + t3 - t2
        del fw, tr
    return d, xt, {"build_s": tb, "fwd_s": tf, "tra_s": tt}


def layer_window_extended(g, kind, consts, layer):
    """Extended-precision (x87 long double, 64-bit significand) response window.

    ACCURACY REFERENCE, not a restatement: the same closed forms as
    :func:`layer_window` evaluated in ``np.longdouble`` (sqrt, log, arctan2
    and every product/sum), then rounded once to float64.  The magnetic
    atan2 sums of deep C4 layers cancel ~1e5-fold, so the reference's fp64
    entries carry ~1e-11 relative error there while these carry ~1e-15: a
    truth against which the reference's own accuracy and the GPU's can both
    be measured (tests/test_gpu_headline.py).
    """
    ld = np.longdouble
    z1, z2 = ld(g.z[layer]), ld(g.z[layer + 1])
    if kind == "gravity":
        cx, cy = corner_vectors(g, "sym")
        q = gravity_corner_sum(z1, z2, cx.astype(ld), cy.astype(ld), ld(consts))
        ax = np.abs(np.arange(g.mx) - (g.sx + g.pxl - 1))
        ay = np.abs(np.arange(g.my) - (g.sy + g.pyl - 1))
        return q[np.ix_(ax, ay)].astype(np.float64)
    cx, cy = corner_vectors(g, "full")
    hx = g.sx + max(g.pxl, g.pxr)
    hy = g.sy + max(g.pyl, g.pyr)
    sx_ = slice(hx - g.sx - g.pxl, hx + g.sx + g.pxr)
    sy_ = slice(hy - g.sy - g.pyl, hy + g.sy + g.pyr)
    w = magnetic_entries(z1, z2, cx[sx_].astype(ld), cy[sy_].astype(ld), np.asarray(consts).astype(ld))
    return w.astype(np.float64)


# --------------------------------------------------------------------------
# independent per-entry dense operator (restates pkg/tests/oracles.py:13-69):
# scalar corner sums with distances recomputed for every station/prism pair,
# no tables, no Toeplitz structure -- a second, structurally different oracle.
# --------------------------------------------------------------------------
def _prism_gravity(x1, x2, y1, y2, z1, z2, gs):
    from math import atan2, log, sqrt
    tot = 0.0
    for i, x in enumerate((x1, x2)):
        for j, y in enumerate((y1, y2)):
            for k, z in enumerate((z1, z2)):
                rho = sqrt(x * x + y * y + z * z)
                tot += (-1.0) ** (i + j + k + 1) * (z * atan2(x * y, z * rho)
                                                    - x * log(rho + y) - y * log(rho + x))
    return gs * tot


def _prism_magnetic(x1, x2, y1, y2, z1, z2, gc):
    from math import atan2, log, sqrt
    tot = 0.0
    for i, x in enumerate((x1, x2)):
        for j, y in enumerate((y1, y2)):
            for k, z in enumerate((z1, z2)):
                rho = sqrt(x * x + y * y + z * z)
                tot += (-1.0) ** (i + j + k + 1) * (
                    gc[0] * log(rho + x) + gc[1] * log(rho + y) + gc[2] * log(rho + z)
                    + gc[3] * atan2(x * z, rho * y) + gc[4] * atan2(y * z, rho * x))
    return tot


def dense_layers(g, kind, consts):
    """Per-layer m x n_r matrices, one scalar kernel call per entry (small grids only)."""
    out = []
    for r in range(g.nz):
        z1, z2 = g.z[r], g.z[r + 1]
        G = np.zeros((g.m, g.n_r))
        for j in range(g.sy):
            b = (g.pyl + j + 0.5) * g.dy
            for i in range(g.sx):
                a = (g.pxl + i + 0.5) * g.dx
                for q in range(g.ny):
                    for p in range(g.nx):
                        args = (p * g.dx - a, (p + 1) * g.dx - a, q * g.dy - b, (q + 1) * g.dy - b, z1, z2)
                        G[j * g.sx + i, q * g.nx + p] = (_prism_gravity(*args, consts) if kind == "gravity"
                                                         else _prism_magnetic(*args, consts))
        out.append(G)
    return out
