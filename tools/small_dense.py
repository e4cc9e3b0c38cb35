"""Single searches on 4 MiB texts (the fused single-wave launch) with dense outputs, event-timed (tools only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for sigma, m in ((2, 2), (2, 4), (4, 2), (4, 4), (16, 2), (1, 2)):
    t = inputs.config2_text(sigma) if sigma > 1 else np.zeros(4 << 20, np.uint8)
    d = torch.from_numpy(t).cuda()
    p = t[1000 : 1000 + m].tobytes()
    pl = engine.Plan(p)
    out = torch.empty(4 << 20, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    l0 = engine.launch_count()
    engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
    nl = engine.launch_count() - l0
    ts = []
    for _ in range(7):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.find_into(pl, d, out, cnt)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    c = int(cnt.item())
    us = sorted(ts)[len(ts) // 2] * 1e3
    print(f"sigma={sigma} m={m} {pl.info().family}: count={c} launches={nl} {us:.1f} us, "
          f"{(t.size + 8 * c) / us / 1e6:.2f} TB/s (n + 8 count)")
