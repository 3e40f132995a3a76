"""Parity on the HEADLINE configuration: C4, all 128 layers, fp64 and fp32.

This is the workload ``bench.py`` times (BASELINE.json configs[3]): 1000 x
1000 stations over 1000 x 1000 x 128 prisms, magnetic kernel D=10, I=60.
The oracle is the reference algorithm (tests' numpy restatement, pinned
bit-identical to the reference) over every layer, threaded over layers with
bounded memory (``O.products_chunked``).  Gates (north_star): rel-L2 <= 1e-10
fp64 and <= 1e-5 fp32, forward and transpose, on

* the bench's own inputs (model U[0, 0.05) from seed 1000 -- rank 0 of
  bench.py -- and data N(0, 1) from seed 1), and
* the survey seeds (model seed 0, data seed 1).

fp32 runs on the fp32-rounded inputs; the oracle is evaluated once, on the
fp64 inputs (input rounding moves the exact products by ~3e-8 relative, far
inside the 1e-5 gate), and both dtypes are checked against it.

Deep layers: G^T of zero-mean data on C4's deepest layers is ill-conditioned
(~1e5-fold cancellation in the magnetic atan2 sums, ~1e3 more in the
product), so the reference's OWN fp64 result there is only good to ~1e-9
(tests/test_reference_conditioning.py).  ``test_deep_layer_transpose_accuracy``
measures both the reference algorithm and the GPU against an extended-
precision truth (entries in x87 long double, ``O.layer_window_extended``) and
requires the GPU to be as accurate as the reference (within 5%) and closer
to the reference than the reference is to the truth.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1912_06976_b200 as B
from oracle import bttb_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-10, "float32": 1e-5}
SEEDS = {"bench": (1000, 1), "survey": (0, 1)}


def _c4():
    og = O.config_grid("C4")
    kind, consts = O.config_kernel("C4")
    sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, _dz, _, kargs, _ = O.CONFIGS["C4"]
    grid = B.make_grid(sx, sy, nz, pxl, pxr, pyl, pyr, dx, dy, og.z)
    return og, kind, consts, grid, B.KernelParams.magnetic(*kargs)


def _inputs(og, which):
    sm, sd = SEEDS[which]
    x = np.random.default_rng(sm).uniform(0.0, 0.05, og.n)
    v = np.random.default_rng(sd).normal(0.0, 1.0, og.m)
    return x, v


@pytest.fixture(scope="module")
def oracle_products():
    cache = {}
    og, kind, consts, _, _ = _c4()

    def get(which):
        if which not in cache:
            x, v = _inputs(og, which)
            with ThreadPoolExecutor(os.cpu_count() or 1) as pool:
                d, xt, _ = O.products_chunked(og, kind, consts, x, v, pool)
            cache[which] = (x, v, d, xt)
        return cache[which]
    return get


@pytest.fixture(scope="module")
def stacks():
    _, _, _, grid, params = _c4()
    out = {dt: B.build_transform_stack(grid, params, dtype=dt) for dt in ("float64", "float32")}
    yield out
    for st in out.values():
        st.close()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("which", ["bench", "survey"])
def test_c4_full_stack_vs_oracle(oracle_products, stacks, which, dtype):
    x, v, d_ref, xt_ref = oracle_products(which)
    st = stacks[dtype]
    assert st.fft_shape == (2048, 2048) and st.nz_local == 128
    f = B.apply(st, x, "forward")
    t = B.apply(st, v, "transpose")
    ef, et = O.rel_l2(d_ref, f), O.rel_l2(xt_ref, t)
    og = O.config_grid("C4")
    per_layer = [O.rel_l2(xt_ref[r * og.n_r:(r + 1) * og.n_r], t[r * og.n_r:(r + 1) * og.n_r])
                 for r in range(og.nz)]
    print(f"C4 x128 {dtype} {which} seeds: forward rel-L2 {ef:.3e}, transpose rel-L2 {et:.3e}; "
          f"per-layer transpose max {max(per_layer):.3e} (layer {int(np.argmax(per_layer))})")
    assert ef <= TOL[dtype]
    assert et <= TOL[dtype]


@pytest.mark.parametrize("layer", [127, 96])
def test_deep_layer_transpose_accuracy(layer):
    """GPU G^T (fp64) on a deep C4 layer is at least as accurate as the
    reference's own fp64 algorithm, both measured against extended precision."""
    og, kind, consts, grid, params = _c4()
    v = np.random.default_rng(1).normal(0.0, 1.0, og.m)

    def tra(window):
        T = O.embed_window(window, og)
        return O.transpose(og, [np.fft.fft2(O.transpose_defining_array(T))], v)

    truth = tra(O.layer_window_extended(og, kind, consts, layer))
    ref = tra(O.layer_window(og, kind, consts, layer))
    with B.build_transform_stack(grid, params, layers=(layer, layer + 1)) as st:
        gpu = B.apply(st, v, "transpose")
    e_ref, e_gpu = O.rel_l2(truth, ref), O.rel_l2(truth, gpu)
    print(f"C4 layer {layer} G^T N(0,1): reference fp64 vs truth {e_ref:.3e}, GPU fp64 vs truth {e_gpu:.3e}, "
          f"GPU vs reference {O.rel_l2(ref, gpu):.3e}")
    # measured (B200, round 2): layer 127 -- reference 1.8289e-8, GPU 1.8290e-8 vs
    # truth, GPU vs reference 3.7e-9.  Both fp64 evaluations share the same
    # IEEE-rounded cancellation of the closed forms (same operation order, so
    # the same rounding); they differ only through libm atan2/log ulps, which
    # is why they are 5x closer to each other than either is to the truth.
    assert e_gpu <= 1.05 * max(e_ref, 1e-12)
    assert O.rel_l2(ref, gpu) <= 0.5 * max(e_ref, 2e-10)
