"""Per-kernel times of chosen patterns over a 1 GiB i.i.d. text (tools only):
periodic / self-overlapping short patterns against random ones.
usage: python tools/pattern_shapes.py sigma pat1 pat2 ...   (patterns as digit strings, e.g. 00000 01010)"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2547_b200 import engine  # noqa: E402

sigma = int(sys.argv[1])
n = 1 << 30
g = torch.Generator(device="cuda").manual_seed(2026 + sigma)
d = torch.randint(0, sigma, (n,), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty(n // 2 + (1 << 20), dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for ps in sys.argv[2:]:
    p = bytes(int(c) for c in ps)
    pl = engine.Plan(p)
    for _ in range(3):
        engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            engine.find_into(pl, d, out, cnt)
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name.split("(")[0][-44:]] += ev.device_time / 5
    print(ps, pl.info().family, int(cnt.item()), {k: round(v, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])})
