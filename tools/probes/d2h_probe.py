"""D2H bandwidth of a 17 GB state into pinned memory: one copy vs chunked copies on k streams."""
import time

import torch

n = 30
x = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
x.fill_(1.0)
h = torch.empty(1 << n, dtype=torch.complex128, pin_memory=True)
torch.cuda.synchronize()
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        chunk = (1 << n) // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i * chunk:(i + 1) * chunk].copy_(x[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{k} streams: {dt * 1e3:.1f} ms, {x.numel() * 16 / dt / 1e9:.1f} GB/s", flush=True)
