"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src; nothing is
copied.  Outputs go to tests/golden/*.npz and are committed so that the CPU
oracle (oracle/bttb_oracle.py) can be pinned on machines without the
reference (the GPU box).  Inputs are regenerated from the same seeds by
oracle.make_inputs / the seeds stored in each file.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import bttb  # noqa: E402  (the reference package)
from bttb.kernels import distance_tables_for, layer_response_window  # noqa: E402

from oracle import bttb_oracle as O  # noqa: E402  (only for the seeded input recipe)

GRAV = bttb.KernelParams.gravity()
MAG = bttb.KernelParams.magnetic(33.0, 47.0, 45000.0)
PADS = [(0, 0, 0, 0), (1, 1, 1, 1), (2, 1, 1, 2), (3, 0, 0, 2)]


def ref_grid(g):
    return bttb.make_grid(g.sx, g.sy, g.nz, g.pxl, g.pxr, g.pyl, g.pyr, g.dx, g.dy, g.z)


def ref_params(name):
    kind, args = O.CONFIGS[name][10], O.CONFIGS[name][11]
    return GRAV if kind == "gravity" else bttb.KernelParams.magnetic(*args)


def small_cases():
    out = {}
    for pads in PADS:
        for params in (GRAV, MAG):
            g = bttb.make_grid(6, 5, 2, *pads, 1.0, 1.5, (0.0, 1.0, 2.5))
            stack = bttb.build_transform_stack(g, params)
            rng = np.random.default_rng(5)
            u = rng.uniform(size=g.n)
            v = rng.uniform(size=g.m)
            tables = distance_tables_for(g, params)
            key = f"{params.kind}_{'_'.join(map(str, pads))}"
            for r in range(g.nz):
                w, _ = layer_response_window(g, tables, params, g.z_blocks[r], g.z_blocks[r + 1])
                out[f"{key}/window{r}"] = w
            out[f"{key}/u"] = u
            out[f"{key}/v"] = v
            out[f"{key}/fwd"] = bttb.apply(stack, u, "forward")
            out[f"{key}/tra"] = bttb.apply(stack, v, "transpose")
    np.savez_compressed(os.path.join(HERE, "small_6x5x2.npz"), **out)


def config_case(name, sub=1):
    g = O.config_grid(name)
    params = ref_params(name)
    rg = ref_grid(g)
    x, d = O.make_inputs(name, g, batch=1)
    stack = bttb.build_transform_stack(rg, params)
    fwd = bttb.apply(stack, x[0], "forward")
    tra = bttb.apply(stack, d[0], "transpose")
    tables = distance_tables_for(rg, params)
    w0, _ = layer_response_window(rg, tables, params, rg.z_blocks[0], rg.z_blocks[1])
    wl, _ = layer_response_window(rg, tables, params, rg.z_blocks[-2], rg.z_blocks[-1])
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), fwd=fwd, tra=tra[::sub], tra_sub=sub,
        tra_norm=np.linalg.norm(tra), window_top=w0, window_bottom=wl,
        x_norm=np.linalg.norm(x), d_norm=np.linalg.norm(d))


def c4_layers():
    """C4 magnetic windows on the top and bottom layers, sampled (full ones are 32 MB)."""
    g = O.config_grid("C4")
    rg = ref_grid(g)
    params = ref_params("C4")
    tables = distance_tables_for(rg, params)
    rng = np.random.default_rng(123)
    ia = rng.integers(0, g.mx, 4096)
    ib = rng.integers(0, g.my, 4096)
    out = {"ia": ia, "ib": ib}
    for r in (0, g.nz - 1):
        w, _ = layer_response_window(rg, tables, params, rg.z_blocks[r], rg.z_blocks[r + 1])
        out[f"w{r}"] = w[ia, ib]
        out[f"w{r}_norm"] = np.linalg.norm(w)
        out[f"w{r}_sum"] = w.sum()
    np.savez_compressed(os.path.join(HERE, "C4_windows.npz"), **out)


def stack_files():
    """Reference-format stack files (the reference's own save_stack) of the
    6x5x2 grid padded (2, 1, 1, 2); products are in small_6x5x2.npz."""
    from bttb.transform import save_stack

    for params in (GRAV, MAG):
        g = bttb.make_grid(6, 5, 2, 2, 1, 1, 2, 1.0, 1.5, (0.0, 1.0, 2.5))
        save_stack(bttb.build_transform_stack(g, params), os.path.join(HERE, f"ref_stack_{params.kind}.bttb"))


if __name__ == "__main__":
    stack_files()
    small_cases()
    config_case("C1")
    config_case("C2")
    config_case("C3", sub=16)
    c4_layers()
    print("golden vectors written to", HERE)
