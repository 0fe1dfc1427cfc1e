"""Pinned host<->device copy bandwidth: H2D, D2H, and both at once (dev tool)."""
import time

import torch

GB = 4 << 30
h_a = torch.empty(GB // 4, dtype=torch.float32).pin_memory()
h_b = torch.empty(GB // 4, dtype=torch.float32).pin_memory()
d_a = torch.empty(GB // 4, dtype=torch.float32, device="cuda")
d_b = torch.empty(GB // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("h2d", "d2h", "both"):
    best = 0
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_a.copy_(h_a, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_b.copy_(d_b, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        gbs = (GB * (2 if name == "both" else 1)) / dt / 1e9
        best = max(best, gbs)
    print(f"{name}: {best:.1f} GB/s (total bytes moved / time)")
print("host cpus", __import__("os").cpu_count())
