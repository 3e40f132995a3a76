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
    reference's count of stored complex values, nz*mx*my).  The per-layer
    full-spectrum tuples ``forward`` / ``transpose`` of the reference are not
    materialised: the device keeps (Hx, Ly) half spectra instead; use
    :meth:`layer_spectrum`.
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
        raise NotImplementedError(
            "the device cache holds (Hx, Ly) half spectra at FFT lengths "
            f"{self.fft_shape}, not the reference's full (mx, my) arrays; "
            "use layer_spectrum()")

    transpose = forward

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
        """GPU-generated response window of a (global) layer, (mx, my) float64."""
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
_KIND_CODES = {"gravity": 0, "magnetic": 1}
_DTYPE_CODES = {"float64": 0, "float32": 1}


def save_stack(stack, path):
    """Persist a device stack: its half spectra as cached, plus what rebuilds the plan.

    Little-endian layout: magic "BTB2" (not the reference's "BTTB": the payload
    is the device cache, (Hx, Ly) half spectra at FFT lengths (Lx, Ly), scaled
    by 1/(Lx*Ly), instead of two full complex128 (mx, my) stacks), version u32,
    kind u8, dtype u8, grid counts 7 x i64, spacings 2 x f64, nz+1 depths,
    gamma*scale f64, gc 5 x f64, kernel D, I, F 3 x f64, layer range 2 x i64,
    Lx, Ly 2 x i64, then layer_end-layer_begin spectra.  Loading gives
    bit-identical products (the spectra are not recomputed).
    """
    g = stack.grid
    p = stack.params
    if p is None:
        raise ValueError("stack has no kernel parameters to persist")
    lx, ly = stack.fft_shape
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack("<IBB", _VERSION, _KIND_CODES[stack.kind], _DTYPE_CODES[str(stack.dtype)]))
        fh.write(struct.pack("<7q", g.sx, g.sy, g.nz, g.pxl, g.pxr, g.pyl, g.pyr))
        fh.write(struct.pack("<2d", g.dx, g.dy))
        fh.write(np.asarray(g.z_blocks, dtype="<f8").tobytes())
        gc = list(p.gc) if p.kind == "magnetic" else [0.0] * 5
        fh.write(struct.pack("<6d", p.gamma * p.scale, *gc))
        fh.write(struct.pack("<3d", p.D, p.I, p.F))
        fh.write(struct.pack("<4q", stack.layer_begin, stack.layer_end, lx, ly))
        for r in range(stack.nz_local):
            fh.write(np.ascontiguousarray(stack.layer_spectrum(r)).tobytes())


def load_stack(path, device=0):
    """Read back a stack written by :func:`save_stack` onto a device (no rebuild)."""
    from .grid import make_grid
    from .kernels import GRAVITATIONAL_CONST, KernelParams

    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic == b"BTTB":
            raise ValueError("reference-format stack file (full complex128 spectra at the "
                             "minimal embedding): rebuild it with build_transform_stack")
        if magic != _MAGIC:
            raise ValueError(f"not a transform-stack file (magic {magic!r})")
        version, kind_code, dt_code = struct.unpack("<IBB", fh.read(6))
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
        hx = lx // 2 + 1
        cdt = np.dtype("<c16" if dtype == "float64" else "<c8")
        count = (hi - lo) * hx * ly
        buf = fh.read(count * cdt.itemsize)
        if len(buf) != count * cdt.itemsize:
            raise ValueError("truncated transform-stack file")
    spectra = np.frombuffer(buf, dtype=cdt)
    if kind == "gravity":
        params = KernelParams(kind="gravity", gamma=GRAVITATIONAL_CONST, scale=gs / GRAVITATIONAL_CONST)
    else:
        params = KernelParams(kind="magnetic", D=D, I=I, F=F, gc=tuple(gc))
    zc = np.ascontiguousarray(grid.z_blocks, dtype=float)
    g = _lib.BttbGrid(grid.sx, grid.sy, grid.nz, grid.pxl, grid.pxr, grid.pyl, grid.pyr,
                      grid.dx, grid.dy, _lib.as_dptr(zc))
    k = params.native()
    if kind == "gravity":
        k.gamma_scaled = gs  # exactly the persisted multiplier
    h = _lib.ctypes.c_void_p()
    _lib.check(_lib.lib().bttb_plan_create_from_spectra(
        _lib.ctypes.byref(h), _lib.ctypes.byref(g), _lib.ctypes.byref(k), _DTYPES[dtype], int(device),
        lo, hi, lx, ly, spectra.ctypes.data_as(_lib.ctypes.c_void_p)))
    return TransformStack(h, grid, kind, dtype, int(device), (lo, hi), 0, params)


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
