"""Build the C4 spectrum cache once (for ncu captures of the entry generator
and the spectrum FFTs; development tool).  python tools/build_step.py [f64|f32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_06976_b200 as B  # noqa: E402
from oracle import bttb_oracle as O  # noqa: E402  (config recipe only)

og = O.config_grid("C4")
sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, dz, _, kargs, _ = O.CONFIGS["C4"]
grid = B.make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, og.z)
dt = "float32" if len(sys.argv) > 1 and sys.argv[1] == "f32" else "float64"
with B.build_transform_stack(grid, B.KernelParams.magnetic(*kargs), dtype=dt) as st:
    print("built", st.fft_shape, st.device_bytes)
