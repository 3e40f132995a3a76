"""Host <-> device copy paths for the reference-API apply (numpy in, numpy out):
1 GB fp64 buffers, pageable vs registered vs pinned staging (development probe)."""
import ctypes
import time

import numpy as np
import torch

n = 128_000_000  # 1.02 GB fp64 (the C4 model vector)
cud = ctypes.CDLL("libcudart.so") if False else None
rt = torch.cuda.cudart()
dev = torch.empty(n, dtype=torch.float64, device="cuda")
x = np.random.default_rng(0).uniform(size=n)


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d_pageable():
    dev.copy_(torch.from_numpy(x))


def h2d_register():
    ptr = x.ctypes.data
    rt.cudaHostRegister(ptr, x.nbytes, 0)
    dev.copy_(torch.from_numpy(x), non_blocking=True)
    torch.cuda.synchronize()
    rt.cudaHostUnregister(ptr)


pin = torch.empty(n, dtype=torch.float64).pin_memory()
pin_np = pin.numpy()


def h2d_staged():
    np.copyto(pin_np, x)
    dev.copy_(pin, non_blocking=True)


def d2h_fresh_pageable():
    out = np.empty(n)
    torch.from_numpy(out).copy_(dev)


def d2h_fresh_pinned():
    out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    return out.numpy()


def d2h_register_fresh():
    out = np.empty(n)
    rt.cudaHostRegister(out.ctypes.data, out.nbytes, 0)
    torch.from_numpy(out).copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    rt.cudaHostUnregister(out.ctypes.data)


def d2h_touched_pageable():
    torch.from_numpy(x).copy_(dev)


for name, f in [("h2d pageable", h2d_pageable), ("h2d register+copy+unregister", h2d_register),
                ("h2d memcpy to pinned + copy", h2d_staged), ("d2h into fresh np.empty", d2h_fresh_pageable),
                ("d2h into touched pageable", d2h_touched_pageable),
                ("d2h into fresh pinned (caching allocator)", d2h_fresh_pinned),
                ("d2h register fresh np.empty", d2h_register_fresh)]:
    print(f"{name:45s} {t(f):8.1f} ms", flush=True)
