"""PCIe D2H rate of one large device->pinned-host copy vs the same bytes split over 2/4 streams
(does the list path's host readback leave bandwidth on the table?). Run under gpurun."""
import time

import torch

GB = 8
n = GB * (1 << 30)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d.fill_(1)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step = n // parts
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"D2H {GB} GiB in {parts} stream(s): {n / best / 1e9:.1f} GB/s")
for parts in (1, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = n // parts
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D {GB} GiB in {parts} stream(s): {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
