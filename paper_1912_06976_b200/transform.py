"""Device-resident spectrum cache: the drop-in for ``build_transform_stack``.

Reference: ``/root/reference/pkg/src/bttb/transform.py``.  The reference keeps,
per layer, the full complex128 fft2 of the circulant embedding T^circ AND of
its transpose layout (2 x mx x my complex per layer, on the host).  Here one
half spectrum per layer is generated and kept in HBM by the sm_100a library
(``bttb_plan_create``):

* entries are generated on the GPU (csrc/entries.cu, kernels.py:81-184);
* the embedding is placed at FFT lengths (Lx, Ly) >= (sx+nx-1, sy+ny-1) with a
  zero gap (same operator);
* the transpose spectrum is conj(forward spectrum) (transform.py:75-82,102), so
  it is not stored;
* the 1/(Lx*Ly) inverse normalisation is folded into the cached spectrum.
"""
import struct
import threading

import numpy as np

from . import _lib
from .grid import GridSpec

__all__ = ["TransformStack", "build_transform_stack", "transpose_layout",
           "circulant_extension_column", "fft_length", "save_stack", "load_stack"]

_DTYPES = {"float64": _lib.F64, "float32": _lib.F32}


def fft_length(n):
    """Smallest FFT length >= n supported by the device FFT engine."""
    return int(_lib.lib().bttb_fft_length(int(n)))


class TransformStack:
    """Handle on a device plan: cached half spectra for layers [layer_begin, layer_end).

    Attributes follow the reference ``TransformStack`` (transform.py:40-58):
    ``grid``, ``kind``, ``kernel_evals_per_layer`` and ``element_count`` (the
    reference's count of stored complex values, nz*mx*my).  The device keeps
    (Hx, Ly) half spectra at FFT lengths ``fft_shape`` (:meth:`layer_spectrum`);
    the reference's full-spectrum tuples ``forward`` / ``transpose`` are
    materialised on the host only when accessed.
    """

    def __init__(self, handle, grid, kind, dtype, device, layer_range, evals, params=None):
        self._handle = handle
        self.params = params
        self._lock = threading.Lock()
        self.grid = grid
        self.kind = kind
        self.dtype = np.dtype(dtype)
        self.device = device
        self.layer_begin, self.layer_end = layer_range
        self.kernel_evals_per_layer = evals
        self._ref_stacks = None
        info = self.info()
        self.fft_shape = (int(info[0]), int(info[1]))
        self.spectrum_shape = (int(info[2]), int(info[1]))

    # -- reference attributes ------------------------------------------------
    @property
    def element_count(self):
        """Complex values the reference would store across its forward stack."""
        mx, my = self.grid.embed_shape
        return self.grid.nz * mx * my

    @property
    def forward(self):
        """Reference-shaped forward stack: per local layer fft2(T^circ), (mx, my) complex128.

        A lazy HOST materialisation for API compatibility (transform.py:40-58,
        :100-101), off the hot path: the GPU-generated window of each layer
        is embedded at the minimal (mx, my) size (transform.py:85-88) and
        transformed with numpy's FFT (lengths like 1999 are outside the device
        FFT family).  Cached after the first access.  The device operator
        never uses it.
        """
        if self._ref_stacks is None:
            self._ref_stacks = _reference_stacks(self)
        return self._ref_stacks[0]

    @property
    def transpose(self):
        """Reference-shaped transpose stack: fft2(transpose_layout(T^circ)) per local layer."""
        if self._ref_stacks is None:
            self._ref_stacks = _reference_stacks(self)
        return self._ref_stacks[1]

    # -- device plan ---------------------------------------------------------
    @property
    def handle(self):
        if self._handle is None:
            raise ValueError("transform stack has been closed")
        return self._handle

    @property
    def nz_local(self):
        return self.layer_end - self.layer_begin

    @property
    def n_local(self):
        return self.grid.n_r * self.nz_local

    @property
    def device_bytes(self):
        hx, ly = self.spectrum_shape
        return self.nz_local * hx * ly * 2 * self.dtype.itemsize

    def info(self):
        buf = (_lib.ctypes.c_int64 * 10)()
        _lib.check(_lib.lib().bttb_plan_info(self.handle, buf))
        return list(buf)

    def layer_spectrum(self, local_layer):
        """Cached half spectrum of a local layer, (Hx, Ly), scaled by 1/(Lx*Ly)."""
        cdt = np.complex128 if self.dtype == np.float64 else np.complex64
        out = np.empty(self.spectrum_shape, dtype=cdt)
        _lib.check(_lib.lib().bttb_layer_spectrum(self.handle, int(local_layer),
                                                  out.ctypes.data_as(_lib.ctypes.c_void_p)))
        return out

    def layer_window(self, layer):
        """Response window of a (global) layer, (mx, my) float64.

        Plans built from kernel constants regenerate it on the GPU
        (``bttb_layer_window``).  Plans loaded from a file carry no kernel
        constants (``params is None``): their window is recovered from the
        cached half spectrum itself (:func:`_window_from_spectrum`), so
        ``forward`` / ``transpose`` / ``save_stack(format="reference")`` of a
        loaded stack reproduce the file's operator.
        """
        if self.params is None:
            if not self.layer_begin <= layer < self.layer_end:
                raise ValueError(f"layer {layer} outside this plan's layers "
                                 f"[{self.layer_begin}, {self.layer_end})")
            return _window_from_spectrum(self.layer_spectrum(layer - self.layer_begin),
                                         self.grid, self.fft_shape)
        out = np.empty(self.grid.embed_shape)
        _lib.check(_lib.lib().bttb_layer_window(self.handle, int(layer), _lib.as_dptr(out)))
        return out

    def close(self):
        h, self._handle = self._handle, None
        if h is not None:
            _lib.lib().bttb_plan_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _evals(grid, kind):
    if kind == "gravity":  # quadrant size, kernels.py:172-174
        return (grid.sx + max(grid.pxl, grid.pxr)) * (grid.sy + max(grid.pyl, grid.pyr))
    mx, my = grid.embed_shape
    return mx * my


def build_transform_stack(grid, params, dtype="float64", device=0, layers=None, fft_shape=None):
    """Generate and cache every layer's spectrum on the GPU (transform.py:91-104).

    Extensions over the reference signature (all optional): ``dtype``
    ("float64" -- reference semantics -- or "float32": fp64 entries and FFT,
    spectra stored and applied in fp32), ``device`` (CUDA ordinal),
    ``layers`` ((begin, end) layer range held by this plan, for layer
    sharding) and ``fft_shape`` ((Lx, Ly) override).
    """
    if not isinstance(grid, GridSpec):
        raise TypeError("grid must be a GridSpec")
    if dtype not in _DTYPES:
        raise ValueError(f"dtype must be one of {sorted(_DTYPES)}, got {dtype!r}")
    lo, hi = (0, grid.nz) if layers is None else (int(layers[0]), int(layers[1]))
    z = np.ascontiguousarray(grid.z_blocks, dtype=float)
    g = _lib.BttbGrid(grid.sx, grid.sy, grid.nz, grid.pxl, grid.pxr, grid.pyl, grid.pyr,
                      grid.dx, grid.dy, _lib.as_dptr(z))
    k = params.native()
    lx, ly = (0, 0) if fft_shape is None else fft_shape
    h = _lib.ctypes.c_void_p()
    _lib.check(_lib.lib().bttb_plan_create(_lib.ctypes.byref(h), _lib.ctypes.byref(g),
                                           _lib.ctypes.byref(k), _DTYPES[dtype], int(device),
                                           lo, hi, int(lx), int(ly)))
    return TransformStack(h, grid, params.kind, dtype, int(device), (lo, hi),
                          _evals(grid, params.kind), params)


# ---------------------------------------------------------------------------
# persistence (transform.py:107-159 of the reference)
# ---------------------------------------------------------------------------
_MAGIC = b"BTB2"
_VERSION = 1
_REF_MAGIC = b"BTTB"  # the reference's own layout (transform.py:19-22)
_REF_VERSION = 1
_KIND_CODES = {"gravity": 0, "magnetic": 1}
_DTYPE_CODES = {"float64": 0, "float32": 1}


def _embedding(window, sx, sy):
    """T^circ of a response window at the minimal size (transform.py:85-88)."""
    return np.roll(window[::-1, ::-1], (sx, sy), axis=(0, 1))


def _window_from_embedding(T, sx, sy):
    """Inverse of :func:`_embedding`: the response window a T^circ holds."""
    return np.roll(T, (-sx, -sy), axis=(0, 1))[::-1, ::-1]


def _window_from_spectrum(S, grid, fft_shape):
    """Response window held by a cached half spectrum (host, off the hot path).

    The plan caches S = fft2(E) / (Lx*Ly), half along x, where E is the
    zero-gap embedding at the FFT lengths: E[t] = h(-pxl-t) for t < sx and
    E[L-u] = h(u-pxl) for 0 < u < nx (per axis; transform.py:85-88 at L >= mx).
    Window entry a holds offset a-(sx+pxl-1), so window[a] = E[sx-1-a] for
    a < sx and window[sx-1+u] = E[L-u].
    """
    lx, ly = fft_shape
    E = np.fft.irfft(np.fft.ifft(np.asarray(S, dtype=np.complex128), axis=1), n=lx, axis=0) * (lx * ly)
    ix = np.concatenate([np.arange(grid.sx - 1, -1, -1), lx - np.arange(1, grid.nx)])
    iy = np.concatenate([np.arange(grid.sy - 1, -1, -1), ly - np.arange(1, grid.ny)])
    return np.ascontiguousarray(E[np.ix_(ix, iy)])


def _reference_stacks(stack):
    fw, tr = [], []
    g = stack.grid
    for r in range(stack.layer_begin, stack.layer_end):
        T = _embedding(stack.layer_window(r), g.sx, g.sy)
        fw.append(np.fft.fft2(T))
        tr.append(np.fft.fft2(transpose_layout(T)))
    return tuple(fw), tuple(tr)


def save_stack(stack, path, format="native"):
    """Persist a stack (transform.py:107-127).

    ``format="native"`` (default): magic "BTB2" -- the device cache itself,
    (Hx, Ly) half spectra at FFT lengths (Lx, Ly) scaled by 1/(Lx*Ly), plus
    what rebuilds the plan.  Little-endian: magic, version u32, kind u8,
    dtype u8, grid counts 7 x i64, spacings 2 x f64, nz+1 depths, gamma*scale
    f64, gc 5 x f64, kernel D, I, F 3 x f64 (NaN when unknown), layer range
    2 x i64, Lx, Ly 2 x i64, then layer_end-layer_begin spectra.  Loading
    gives bit-identical products (nothing is recomputed).

    ``format="reference"``: the reference's own "BTTB" v1 layout (full
    complex128 fft2 of T^circ and of its transpose layout at (mx, my), every
    layer), readable by the reference's ``load_stack``.  Written from the
    GPU-generated windows through :attr:`TransformStack.forward`; needs a plan
    holding all nz layers.
    """
    if format == "reference":
        return _save_reference(stack, path)
    if format != "native":
        raise ValueError(f"format must be 'native' or 'reference', got {format!r}")
    g = stack.grid
    p = stack.params
    lx, ly = stack.fft_shape
    nan = float("nan")
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack("<IBB", _VERSION, _KIND_CODES[stack.kind], _DTYPE_CODES[str(stack.dtype)]))
        fh.write(struct.pack("<7q", g.sx, g.sy, g.nz, g.pxl, g.pxr, g.pyl, g.pyr))
        fh.write(struct.pack("<2d", g.dx, g.dy))
        fh.write(np.asarray(g.z_blocks, dtype="<f8").tobytes())
        if p is None:
            fh.write(struct.pack("<6d", *([nan] * 6)))
            fh.write(struct.pack("<3d", nan, nan, nan))
        else:
            gc = list(p.gc) if p.kind == "magnetic" else [0.0] * 5
            fh.write(struct.pack("<6d", p.gamma * p.scale, *gc))
            fh.write(struct.pack("<3d", p.D, p.I, p.F))
        fh.write(struct.pack("<4q", stack.layer_begin, stack.layer_end, lx, ly))
        for r in range(stack.nz_local):
            fh.write(np.ascontiguousarray(stack.layer_spectrum(r)).tobytes())


def _save_reference(stack, path):
    g = stack.grid
    if (stack.layer_begin, stack.layer_end) != (0, g.nz):
        raise ValueError("the reference stack format holds every layer; this plan holds layers "
                         f"[{stack.layer_begin}, {stack.layer_end}) of {g.nz}")
    mx, my = g.embed_shape
    with open(path, "wb") as fh:
        fh.write(_REF_MAGIC)
        fh.write(struct.pack("<IB", _REF_VERSION, _KIND_CODES[stack.kind]))
        fh.write(struct.pack("<7q", g.sx, g.sy, g.nz, g.pxl, g.pxr, g.pyl, g.pyr))
        fh.write(struct.pack("<2d", g.dx, g.dy))
        fh.write(np.asarray(g.z_blocks, dtype="<f8").tobytes())
        fh.write(struct.pack("<3q", g.nz, mx, my))
        for arr in stack.forward + stack.transpose:
            fh.write(np.ascontiguousarray(arr, dtype="<c16").tobytes())


def _native_params(kind, gs, gc, D, I, F):  # noqa: E741
    from .kernels import GRAVITATIONAL_CONST, KernelParams

    if not np.isfinite(gs):
        return None
    if kind == "gravity":
        return KernelParams(kind="gravity", gamma=GRAVITATIONAL_CONST, scale=gs / GRAVITATIONAL_CONST)
    return KernelParams(kind="magnetic", D=D, I=I, F=F, gc=tuple(gc))


def _grid_struct(grid):
    zc = np.ascontiguousarray(grid.z_blocks, dtype=float)
    return _lib.BttbGrid(grid.sx, grid.sy, grid.nz, grid.pxl, grid.pxr, grid.pyl, grid.pyr,
                         grid.dx, grid.dy, _lib.as_dptr(zc)), zc


def load_stack(path, device=0, dtype=None):
    """Read back a persisted stack onto a device (transform.py:130-159).

    Native "BTB2" files upload their cached spectra (no rebuild; ``dtype``
    must be None or the file's).  Reference "BTTB" files (the reference's
    ``save_stack`` output) are accepted too: each layer's T^circ is recovered
    on the host as real(ifft2(forward[r])) -- a format conversion, off the
    hot path -- and the GPU rebuilds the spectra from those windows
    (``bttb_plan_create_from_windows``) at the plan's FFT lengths, in
    ``dtype`` (default "float64").  Error messages follow the reference
    ("magic", "unsupported stack version", "inconsistent", "truncated").
    """
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic == _REF_MAGIC:
            return _load_reference(fh, device, dtype or "float64")
        if magic != _MAGIC:
            raise ValueError(f"not a transform-stack file (magic {magic!r})")
        return _load_native(fh, device, dtype)


def _load_native(fh, device, want_dtype):
    from .grid import make_grid

    head = fh.read(6)
    if len(head) != 6:
        raise ValueError("truncated transform-stack file")
    version, kind_code, dt_code = struct.unpack("<IBB", head)
    if version != _VERSION:
        raise ValueError(f"unsupported stack version {version}")
    sx, sy, nz, pxl, pxr, pyl, pyr = struct.unpack("<7q", fh.read(56))
    dx, dy = struct.unpack("<2d", fh.read(16))
    z = np.frombuffer(fh.read(8 * (nz + 1)), dtype="<f8")
    gs, *gc = struct.unpack("<6d", fh.read(48))
    D, I, F = struct.unpack("<3d", fh.read(24))  # noqa: E741
    lo, hi, lx, ly = struct.unpack("<4q", fh.read(32))
    grid = make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, z)
    kind = {0: "gravity", 1: "magnetic"}[kind_code]
    dtype = {0: "float64", 1: "float32"}[dt_code]
    if want_dtype is not None and want_dtype != dtype:
        raise ValueError(f"stack file holds {dtype} spectra, {want_dtype} requested")
    hx = lx // 2 + 1
    cdt = np.dtype("<c16" if dtype == "float64" else "<c8")
    count = (hi - lo) * hx * ly
    buf = fh.read(count * cdt.itemsize)
    if len(buf) != count * cdt.itemsize:
        raise ValueError("truncated transform-stack file")
    spectra = np.frombuffer(buf, dtype=cdt)
    params = _native_params(kind, gs, gc, D, I, F)
    g, _z = _grid_struct(grid)
    k = _lib.BttbKernel(_lib.GRAVITY if kind == "gravity" else _lib.MAGNETIC,
                        gs if np.isfinite(gs) else 0.0, (_lib.ctypes.c_double * 5)(*gc))
    h = _lib.ctypes.c_void_p()
    _lib.check(_lib.lib().bttb_plan_create_from_spectra(
        _lib.ctypes.byref(h), _lib.ctypes.byref(g), _lib.ctypes.byref(k), _DTYPES[dtype], int(device),
        lo, hi, lx, ly, spectra.ctypes.data_as(_lib.ctypes.c_void_p)))
    return TransformStack(h, grid, kind, dtype, int(device), (lo, hi), 0, params)


def _load_reference(fh, device, dtype):
    from .grid import make_grid

    if dtype not in _DTYPES:
        raise ValueError(f"dtype must be one of {sorted(_DTYPES)}, got {dtype!r}")
    head = fh.read(5)
    if len(head) != 5:
        raise ValueError("truncated transform-stack file")
    version, kind_code = struct.unpack("<IB", head)
    if version != _REF_VERSION:
        raise ValueError(f"unsupported stack version {version}")
    if kind_code not in (0, 1):
        raise ValueError(f"unknown kernel kind code {kind_code}")
    sx, sy, nz, pxl, pxr, pyl, pyr = struct.unpack("<7q", fh.read(56))
    dx, dy = struct.unpack("<2d", fh.read(16))
    z = np.frombuffer(fh.read(8 * (nz + 1)), dtype="<f8")
    layers, mx, my = struct.unpack("<3q", fh.read(24))
    grid = make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, z)
    if (mx, my) != grid.embed_shape or layers != nz:
        raise ValueError("stack header is inconsistent with its grid")
    count = mx * my
    windows = np.empty((nz, mx, my))
    for r in range(nz):
        buf = fh.read(16 * count)
        if len(buf) != 16 * count:
            raise ValueError("truncated transform-stack file")
        F = np.frombuffer(buf, dtype="<c16").reshape(mx, my)
        windows[r] = _window_from_embedding(np.fft.ifft2(F).real, sx, sy)
    # the transpose stack is conj(forward) for a real T^circ; it is read only
    # to keep the reference's truncation semantics
    for _ in range(nz):
        if len(fh.read(16 * count)) != 16 * count:
            raise ValueError("truncated transform-stack file")
    kind = {0: "gravity", 1: "magnetic"}[kind_code]
    g, _z = _grid_struct(grid)
    k = _lib.BttbKernel(_lib.GRAVITY if kind == "gravity" else _lib.MAGNETIC, 0.0,
                        (_lib.ctypes.c_double * 5)())
    h = _lib.ctypes.c_void_p()
    _lib.check(_lib.lib().bttb_plan_create_from_windows(
        _lib.ctypes.byref(h), _lib.ctypes.byref(g), _lib.ctypes.byref(k), _DTYPES[dtype], int(device),
        0, nz, 0, 0, _lib.as_dptr(windows)))
    return TransformStack(h, grid, kind, dtype, int(device), (0, nz), 0, None)


def transpose_layout(T):
    """Defining array of the transposed BCCB: T~[t] = T[-t] (transform.py:75-82).

    Host layout helper kept for API compatibility; the device path never forms
    it (the transpose spectrum is the conjugate of the forward one).
    """
    T = np.asarray(T)
    return np.roll(np.flip(T, (0, 1)), 1, axis=(0, 1))


def circulant_extension_column(c, r):
    """(c; reverse(r[1:])): first column of the circulant extending toeplitz(c, r)."""
    c = np.asarray(c, dtype=float)
    r = np.asarray(r, dtype=float)
    if c[0] != r[0]:
        raise ValueError(
            f"c[0] and r[0] must be the shared corner element, got {c[0]} != {r[0]}")
    return np.concatenate([c, r[1:][::-1]])
