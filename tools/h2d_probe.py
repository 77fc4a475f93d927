"""Pinned host -> HBM copy bandwidth with 1, 2 and 4 concurrent streams (1 GiB)."""
import time
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams={k}: {n / dt / 1e9:.1f} GB/s")
