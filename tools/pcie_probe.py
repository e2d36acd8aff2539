"""Pinned host<->device copy bandwidth on this box (the e2e ceiling):
one-direction and both directions at once, 822 MB (cfg2's y) and 154 MB (x)."""
import time
import torch

dev = torch.device("cuda", 0)
for mb in (154, 822):
    n = mb * 1024 * 1024 // 4
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)),
                     ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"{name} {mb} MB: {mb * 1.048576e6 / dt / 1e9:.1f} GB/s")
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"both {mb} MB each way: {2 * mb * 1.048576e6 / dt / 1e9:.1f} GB/s total")
