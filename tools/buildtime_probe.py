import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1912_06976_b200 as B
GRAV = B.KernelParams.gravity()
for rep in range(3):
    for k in (2, 3, 4):
        g = B.scaled_problem(k, 0.0)
        B.build_transform_stack(g, GRAV).close()
        t0 = time.perf_counter(); st = B.build_transform_stack(g, GRAV); t = time.perf_counter() - t0
        u = np.random.default_rng(0).uniform(size=g.n)
        B.apply(st, u, "forward")
        t1 = time.perf_counter(); B.apply(st, u, "forward"); t2 = time.perf_counter() - t1
        print(rep, k, st.fft_shape, f"build {t*1e3:.2f} ms fwd {t2*1e3:.3f} ms", flush=True)
        st.close()
