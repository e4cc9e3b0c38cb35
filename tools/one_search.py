"""Repeat one single-pattern search on a seeded i.i.d. text (for ncu captures).
usage: python tools/one_search.py sigma m [family] [MiB] [reps]   (tools only)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2547_b200 import engine  # noqa: E402

sigma, m = int(sys.argv[1]), int(sys.argv[2])
fam = sys.argv[3] if len(sys.argv) > 3 else "auto"
n = (int(sys.argv[4]) if len(sys.argv) > 4 else 1024) << 20
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
g = torch.Generator(device="cuda").manual_seed(2026 + sigma)
d = torch.randint(0, sigma, (n,), dtype=torch.uint8, device="cuda", generator=g)
pl = engine.Plan(d[n // 3 + 17 * m : n // 3 + 18 * m].cpu().numpy().tobytes(), fam)
out = torch.empty(n // 4 + (1 << 20), dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(reps):
    engine.find_into(pl, d, out, cnt)
torch.cuda.synchronize()
print(sigma, m, pl.info(), int(cnt.item()))
