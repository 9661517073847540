"""Pinned host<->device copy bandwidth on the GPU box (context for e2e)."""
import time
import torch
for mb in (128, 571):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"{name} {mb} MiB: {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms)")
