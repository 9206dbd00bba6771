"""Pinned host->device bandwidth on the box (context for the e2e upload phase)."""
import time
import torch
for mb in (8, 64, 168):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(f"H2D {mb} MiB: {dt*1e3:.3f} ms, {(mb << 20)/dt/1e9:.1f} GB/s")
