"""Per-kernel device times of single-pattern searches on a 1 GiB i.i.d. text
(torch.profiler CUPTI records: real clocks, no replay).  Tools only.

usage: python tools/cell_kernels.py sigma:m[:family] [sigma:m ...]
"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2547_b200 import engine  # noqa: E402

n = 1 << 30
texts = {}
out = torch.empty(n // 4 + (1 << 20), dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for spec in sys.argv[1:]:
    parts = spec.split(":")
    sigma, m = int(parts[0]), int(parts[1])
    fam = parts[2] if len(parts) > 2 else "auto"
    if sigma not in texts:
        g = torch.Generator(device="cuda").manual_seed(2026 + sigma)
        texts[sigma] = torch.randint(0, sigma, (n,), dtype=torch.uint8, device="cuda", generator=g)
    d = texts[sigma]
    off = n // 3 + 17 * m
    pl = engine.Plan(d[off : off + m].cpu().numpy().tobytes(), fam)
    for _ in range(3):
        engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
    reps = 5
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            engine.find_into(pl, d, out, cnt)
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name] += ev.device_time / reps
    tot = sum(agg.values())
    inf = pl.info()
    print(f"sigma={sigma} m={m} family={inf.family} words={inf.words} count={int(cnt.item())} "
          f"kernels={tot:.1f} us")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"   {v:9.1f} us  {k[:110]}")
