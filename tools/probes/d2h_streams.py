"""D2H bandwidth of a 16 GB state into pinned host memory: one copy vs chunks on 2 / 4 / 8
streams (copy engines)."""
import time

import torch

n = 30
src = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
dst = torch.empty(1 << n, dtype=torch.complex128, pin_memory=True)
for k in (1, 2, 4, 8, 1):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = (1 << n) // k
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{k} streams: {dt * 1e3:.1f} ms, {src.numel() * 16 / dt / 1e9:.1f} GB/s", flush=True)
for k in (1, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = (1 << n) // k
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            src[i * chunk:(i + 1) * chunk].copy_(dst[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"H2D {k} streams: {dt * 1e3:.1f} ms, {src.numel() * 16 / dt / 1e9:.1f} GB/s", flush=True)
