"""Kernel constants (host) and the GPU kernel-entry generator front end.

Mirrors ``/root/reference/pkg/src/bttb/kernels.py``.  ``KernelParams`` and
``magnetic_constants`` are five-number parameter setup done on the host (the
same numpy expressions as kernels.py:48-64, so the constants handed to the
device are bit-identical).  The entries themselves -- ``gravity_layer_response``,
``magnetic_response`` and ``layer_response_window`` -- are evaluated by the
sm_100a entry generators in ``csrc/entries.cu`` through the C ABI.
"""
from dataclasses import dataclass

import numpy as np

from . import _lib
from .grid import full_distances, sym_distances

__all__ = ["GRAVITATIONAL_CONST", "KernelParams", "magnetic_constants",
           "gravity_layer_response", "magnetic_response", "layer_response_window",
           "distance_tables_for"]

#: CODATA gravitational constant, m^3 kg^-1 s^-2 (kernels.py:16).
GRAVITATIONAL_CONST = 6.67430e-11


@dataclass(frozen=True)
class KernelParams:
    """Kernel selection plus constants (kernels.py:19-45)."""

    kind: str
    gamma: float = GRAVITATIONAL_CONST
    scale: float = 1.0
    D: float = 0.0
    I: float = 90.0  # noqa: E741
    F: float = 50000.0
    gc: tuple = ()

    @classmethod
    def gravity(cls, gamma=GRAVITATIONAL_CONST, scale=1.0):
        if not gamma > 0:
            raise ValueError(f"gamma must be positive, got {gamma}")
        return cls(kind="gravity", gamma=gamma, scale=scale)

    @classmethod
    def magnetic(cls, D, I, F):  # noqa: E741
        return cls(kind="magnetic", D=float(D), I=float(I), F=float(F),
                   gc=tuple(magnetic_constants(D, I, F)))

    def native(self):
        """The C-ABI kernel record (gamma*scale, kernels.py:98; gc, kernels.py:152)."""
        k = _lib.BttbKernel()
        if self.kind == "gravity":
            k.kind = _lib.GRAVITY
            k.gamma_scaled = self.gamma * self.scale
        elif self.kind == "magnetic":
            k.kind = _lib.MAGNETIC
            for i, g in enumerate(self.gc):
                k.gc[i] = g
        else:
            raise ValueError(f"unknown kernel kind {self.kind!r}")
        return k


def magnetic_constants(D, I, F):  # noqa: E741
    """(2mn, 2ln, 2lm, n^2-m^2, n^2-l^2) * F/(4 pi); x North, y East, z down."""
    if not F > 0:
        raise ValueError(f"F must be positive, got {F}")
    d, i = np.radians(D), np.radians(I)
    cl = np.cos(i) * np.cos(d)
    cm = np.cos(i) * np.sin(d)
    cn = np.sin(i)
    return (F / (4.0 * np.pi)) * np.array(
        [2 * cm * cn, 2 * cl * cn, 2 * cl * cm, cn * cn - cm * cm, cn * cn - cl * cl])


def _depths(z1, z2):
    if z2 < z1:
        raise ValueError(f"layer depths must satisfy z2 >= z1, got ({z1}, {z2})")
    if z1 < 0:
        raise ValueError(f"layer top must satisfy z1 >= 0, got {z1}")
    return float(z1), float(z2)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=float))


def gravity_layer_response(z1, z2, tables, params, device=0):
    """Vertical-gravity entries over a corner table, on the GPU (kernels.py:81-102)."""
    z1, z2 = _depths(z1, z2)
    x, y = _f64(tables.x), _f64(tables.y)
    xy, r2 = _f64(tables.xy), _f64(tables.r2)
    out = np.empty((x.size - 1, y.size - 1))
    if out.size:
        _lib.check(_lib.lib().bttb_gravity_response(
            _lib.as_dptr(x), x.size, _lib.as_dptr(y), y.size, _lib.as_dptr(xy), _lib.as_dptr(r2),
            z1, z2, params.gamma * params.scale, _lib.as_dptr(out), device))
    return out


def magnetic_response(z1, z2, X, Y, R2, gc, device=0):
    """Total-field entries over a corner table, on the GPU (kernels.py:105-155)."""
    z1, z2 = _depths(z1, z2)
    x, y, r2 = _f64(X), _f64(Y), _f64(R2)
    g = _f64(gc)
    out = np.empty((x.size - 1, y.size - 1))
    if out.size:
        _lib.check(_lib.lib().bttb_magnetic_response(
            _lib.as_dptr(x), x.size, _lib.as_dptr(y), y.size, _lib.as_dptr(r2), z1, z2,
            _lib.as_dptr(g), _lib.as_dptr(out), device))
    return out


def layer_response_window(grid, tables, params, z1, z2, device=0):
    """Response at every signed offset the layer needs (kernels.py:158-184).

    Returns (window, evaluation_count); entry (a, b) is offset
    (a-(sx+pxl-1), b-(sy+pyl-1)).  Gravity is evaluated on the quadrant and
    mirrored by |offset|, magnetic on the full window.
    """
    mx, my = grid.embed_shape
    if params.kind == "gravity":
        if tables.flavor != "sym":
            raise ValueError("gravity window needs sym-flavor distance tables")
        quad = gravity_layer_response(z1, z2, tables, params, device)
        ia = np.abs(np.arange(mx) - (grid.sx + grid.pxl - 1))
        ib = np.abs(np.arange(my) - (grid.sy + grid.pyl - 1))
        return quad[np.ix_(ia, ib)], quad.size
    if tables.flavor != "full":
        raise ValueError("magnetic window needs full-flavor distance tables")
    hx = grid.sx + max(grid.pxl, grid.pxr)
    hy = grid.sy + max(grid.pyl, grid.pyr)
    sa = slice(hx - grid.sx - grid.pxl, hx + grid.sx + grid.pxr)
    sb = slice(hy - grid.sy - grid.pyl, hy + grid.sy + grid.pyr)
    win = magnetic_response(z1, z2, tables.x[sa], tables.y[sb], tables.r2[sa, sb],
                            params.gc, device)
    return win, win.size


def distance_tables_for(grid, params):
    """sym tables for gravity, full tables otherwise (kernels.py:187-191)."""
    return sym_distances(grid) if params.kind == "gravity" else full_distances(grid)
