"""Device timeline (CUPTI via torch.profiler) of one prepared config-2 batch (tools only).
usage: batch_timeline.py SIGMA M"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

sigma, m = int(sys.argv[1]), int(sys.argv[2])
t = inputs.config2_text(sigma)
d = torch.from_numpy(t).cuda()
b = engine.Batch([engine.Plan(p) for p in inputs.config2_patterns(t, sigma, m)])
offs = torch.zeros(len(b) + 1, dtype=torch.int64, device="cuda")
engine.find_batch_into(b, d, None, offs)
out = torch.empty(max(int(offs[-1]), 1), dtype=torch.int64, device="cuda")
for _ in range(3):
    engine.find_batch_into(b, d, out, offs)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch.cuda._sleep(2_000_000)
    engine.find_batch_into(b, d, out, offs)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.end
for e in evs[1:]:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:70]}")
