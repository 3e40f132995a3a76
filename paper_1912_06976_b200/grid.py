"""Survey geometry (host side): padded prism grids and staggered distances.

Mirrors ``/root/reference/pkg/src/bttb/grid.py`` (same names, fields, derived
sizes and ValueError messages) so callers can switch packages unchanged.  This
module is plain host bookkeeping; the distance arithmetic that feeds the kernel
entries is redone bit-identically on the device (csrc/capi.cu
``corner_vectors``), the tables here exist for API compatibility.
"""
from dataclasses import dataclass

import numpy as np

__all__ = ["GridSpec", "make_grid", "scaled_problem", "DistanceTables",
           "sym_distances", "full_distances"]


def _int_field(name, value, minimum):
    ok = isinstance(value, (int, np.integer)) and not isinstance(value, bool) and value >= minimum
    if not ok:
        kind = "a positive" if minimum == 1 else "a non-negative"
        raise ValueError(f"{name} must be {kind} integer, got {value!r}")
    return int(value)


@dataclass(frozen=True)
class GridSpec:
    """Station counts, per-side padding, spacings and depth coordinates.

    Same contract as the reference ``GridSpec`` (grid.py:26-104): ``nx = sx +
    pxl + pxr``, ``ny`` likewise, ``m = sx*sy``, ``n_r = nx*ny``, ``n = n_r*nz``
    and ``embed_shape = (sx+nx-1, sy+ny-1)``.
    """

    sx: int
    sy: int
    nz: int
    pxl: int
    pxr: int
    pyl: int
    pyr: int
    dx: float
    dy: float
    z_blocks: tuple

    def __post_init__(self):
        set_ = object.__setattr__
        for name in ("sx", "sy", "nz"):
            set_(self, name, _int_field(name, getattr(self, name), 1))
        for name in ("pxl", "pxr", "pyl", "pyr"):
            set_(self, name, _int_field(name, getattr(self, name), 0))
        for name in ("dx", "dy"):
            val = float(getattr(self, name))
            if not val > 0.0:
                raise ValueError(f"{name} must be positive, got {val}")
            set_(self, name, val)
        depths = tuple(float(z) for z in self.z_blocks)
        if len(depths) != self.nz + 1:
            raise ValueError(
                f"z_blocks must have nz+1={self.nz + 1} entries, got {len(depths)}")
        if depths[0] < 0.0:
            raise ValueError(f"z_blocks[0] must be >= 0, got {depths[0]}")
        if any(lo >= hi for lo, hi in zip(depths[:-1], depths[1:])):
            raise ValueError(f"z_blocks must be strictly increasing, got {depths}")
        set_(self, "z_blocks", depths)

    nx = property(lambda self: self.sx + self.pxl + self.pxr)
    ny = property(lambda self: self.sy + self.pyl + self.pyr)
    m = property(lambda self: self.sx * self.sy, doc="Number of stations.")
    n_r = property(lambda self: self.nx * self.ny, doc="Prisms per depth layer.")
    n = property(lambda self: self.n_r * self.nz, doc="Total number of prisms.")

    @property
    def embed_shape(self):
        """Minimal circulant-embedding shape of one layer (the reference's)."""
        return (self.sx + self.nx - 1, self.sy + self.ny - 1)


def make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, z_blocks):
    """Validated :class:`GridSpec` (grid.py:107-116)."""
    return GridSpec(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, tuple(z_blocks))


def scaled_problem(k, pad_fraction, dx=100.0, dy=100.0, dz=100.0):
    """Benchmark family member k: (25k, 15k) stations, 2k layers (grid.py:124-147).

    Per-side padding rounds pad_fraction*s half away from zero.
    """
    k = _int_field("k", k, 1)
    if pad_fraction < 0:
        raise ValueError(f"pad_fraction must be >= 0, got {pad_fraction}")
    sx, sy, nz = 25 * k, 15 * k, 2 * k
    px = int(np.floor(pad_fraction * sx + 0.5))
    py = int(np.floor(pad_fraction * sy + 0.5))
    return make_grid(sx, sy, nz, px, px, py, py, dx, dy, [r * dz for r in range(nz + 1)])


@dataclass(frozen=True)
class DistanceTables:
    """Corner distance vectors x, y with xy = x (x) y and r2 = x^2 + y^2."""

    x: np.ndarray
    y: np.ndarray
    xy: np.ndarray
    r2: np.ndarray
    flavor: str

    def __post_init__(self):
        for arr in (self.x, self.y, self.xy, self.r2):
            arr.flags.writeable = False


def _tables(x, y, flavor):
    return DistanceTables(x=x, y=y, xy=np.multiply.outer(x, y),
                          r2=np.add.outer(x ** 2, y ** 2), flavor=flavor)


def sym_distances(grid):
    """First-station corner distances (l - 1/2)*d, l = 0..s+max(pad) (grid.py:177-187)."""
    hx = grid.sx + max(grid.pxl, grid.pxr)
    hy = grid.sy + max(grid.pyl, grid.pyr)
    return _tables((np.arange(hx + 1) - 0.5) * grid.dx,
                   (np.arange(hy + 1) - 0.5) * grid.dy, "sym")


def full_distances(grid):
    """All station/corner offsets, 2*(s+max(pad)) per axis (grid.py:190-199)."""
    hx = grid.sx + max(grid.pxl, grid.pxr)
    hy = grid.sy + max(grid.pyl, grid.pyr)
    return _tables((np.arange(2 * hx) - hx + 0.5) * grid.dx,
                   (np.arange(2 * hy) - hy + 0.5) * grid.dy, "full")
