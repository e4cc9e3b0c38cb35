"""Device timeline (CUPTI via torch.profiler) of one config-5 search (tools only).
usage: cfg5_timeline.py M am|amb"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

m, kind = int(sys.argv[1]), sys.argv[2]
t = inputs.config5()
d = torch.from_numpy(t).cuda()
pl = engine.Plan(b"a" * m if kind == "am" else b"a" * (m - 1) + b"b")
c = engine.count(pl, d)
out = torch.empty(max(c, 1), dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    engine.find_into(pl, d, out, cnt)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch.cuda._sleep(2_000_000)
    engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.end
for e in evs[1:]:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:70]}")
