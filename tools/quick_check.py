"""Quick GPU parity probe against the oracle (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

def run(name, g, kind, consts, params, dtype="float64", nz_batch=None):
    t0 = time.time()
    fw, tr = O.build_spectra(g, kind, consts)
    rng = np.random.default_rng(5)
    u = rng.uniform(size=g.n); v = rng.uniform(size=g.m)
    fo = O.forward(g, fw, u); to = O.transpose(g, tr, v)
    bg = B.make_grid(g.sx, g.sy, g.nz, g.pxl, g.pxr, g.pyl, g.pyr, g.dx, g.dy, g.z)
    st = B.build_transform_stack(bg, params, dtype=dtype)
    w0 = st.layer_window(0); wo = O.layer_window(g, kind, consts, 0)
    fg = B.apply(st, u, "forward"); tg = B.apply(st, v, "transpose")
    print(f"{name:28s} {dtype} L={st.fft_shape} win0 {np.abs(w0-wo).max()/np.abs(wo).max():.2e} "
          f"fwd {O.rel_l2(fo, fg):.2e} tra {O.rel_l2(to, tg):.2e}  ({time.time()-t0:.1f}s)", flush=True)

GRAV = B.KernelParams.gravity(); MAG = B.KernelParams.magnetic(33.0, 47.0, 45000.0)
for pads in [(0,0,0,0),(1,1,1,1),(2,1,1,2),(3,0,0,2)]:
    g = O.ogrid(6,5,2,*pads,1.0,1.5,(0.0,1.0,2.5))
    run(f"6x5x2 {pads} grav", g, "gravity", O.grav_constants(), GRAV)
    run(f"6x5x2 {pads} mag", g, "magnetic", O.mag_constants(33.,47.,45000.), MAG)
for name in ["C1", "C2", "C3"]:
    g = O.config_grid(name); kind, c = O.config_kernel(name)
    p = GRAV if kind == "gravity" else B.KernelParams.magnetic(*O.CONFIGS[name][11])
    run(name, g, kind, c, p)
    run(name, g, kind, c, p, "float32")
# C4 geometry, 3 layers (TMA column path at L=2000), fp64 and fp32
g = O.config_grid("C4", nz=3); kind, c = O.config_kernel("C4")
p = B.KernelParams.magnetic(*O.CONFIGS["C4"][11])
run("C4[3 layers]", g, kind, c, p)
run("C4[3 layers]", g, kind, c, p, "float32")
