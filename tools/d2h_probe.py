"""D2H bandwidth probe: pinned destination, 1 vs 2 vs 4 concurrent streams."""
import time

import torch

n = 38 << 20
src = torch.empty(n, dtype=torch.uint8, device="cuda").random_(0, 255)
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"streams={k}: {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.3f} ms)", flush=True)
h2d_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(h2d_src, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"H2D: {n / dt / 1e9:.1f} GB/s")
