"""Concurrent pinned H2D + D2H of 1.03 GB each (the e2e step's copy pattern)."""
import time
import torch
n = 129_000_000
a = torch.empty(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
da = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.zeros(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d=True, d2h=True):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3):
        if h2d:
            with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / 3 * 1e3
run()
print(f"h2d alone {run(True, False):.1f} ms, d2h alone {run(False, True):.1f} ms, both {run():.1f} ms per 1.03 GB each")
