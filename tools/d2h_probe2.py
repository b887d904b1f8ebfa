"""D2H bandwidth of one 38 MB pinned copy vs the same bytes split over two
or four streams (copy engines), and vs chunked copies on one stream."""
import time

import torch

n = 38 << 20
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
dev.random_(0, 255)
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(4)]


def run(parts, nstreams, reps=20):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for j in range(parts):
            a, b = n * j // parts, n * (j + 1) // parts
            with torch.cuda.stream(streams[j % nstreams]):
                host[a:b].copy_(dev[a:b], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    ts = sorted(ts)[2:-2]
    return n / (sum(ts) / len(ts)) / 1e9


for parts, ns in ((1, 1), (2, 2), (4, 4), (4, 1), (8, 2), (16, 4)):
    print(f"parts={parts} streams={ns}: {run(parts, ns):.1f} GB/s", flush=True)
