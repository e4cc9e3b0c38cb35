"""H2D bandwidth of a pinned 16 GiB buffer: one copy vs chunked copies on 1-4 streams (tools only)."""
import time

import torch

n = 16 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(7)
d = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(nstreams, chunk):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    i = 0
    for off in range(0, n, chunk):
        s = streams[i % nstreams]
        with torch.cuda.stream(s):
            d[off : off + chunk].copy_(h[off : off + chunk], non_blocking=True)
        i += 1
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"streams={nstreams} chunk={chunk >> 20} MiB: {n / dt / 1e9:.1f} GB/s", flush=True)


for ns, ch in [(1, n), (1, 256 << 20), (2, 256 << 20), (4, 256 << 20), (2, 1 << 30), (4, 64 << 20)]:
    run(ns, ch)
