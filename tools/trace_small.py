"""Kernel start/end timeline of a few small searches (CUPTI via torch.profiler; tools only)."""
import sys, torch
sys.path.insert(0, '.')
from torch.profiler import profile, ProfilerActivity
from paper_1012_2547_b200 import engine, inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
t = inputs.rand_text_np(4, n, 3); d = torch.from_numpy(t).cuda()
pl = engine.Plan(t[1000:1008].tobytes())
out = torch.empty(1 << 16, dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(5): engine.find_into(pl, d, out, cnt)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch.cuda._sleep(2_000_000)
    for _ in range(3): engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:60]}")
