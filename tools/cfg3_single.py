"""One config-3 single-pattern search (m) on the 64 MiB Zipf text, timed (tools only)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

m = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t = inputs.config3()
d = torch.from_numpy(t).cuda()
p = inputs.config3_patterns(t, m)[0]
pl = engine.Plan(p)
out = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(400_000)
    e0.record()
    engine.find_into(pl, d, out, cnt)
    e1.record()
    torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1) * 1e3, 1))
inf = pl.info()
print(m, inf.family, "stride", inf.stride, "gram", inf.gram, "count", int(cnt.item()), "us", ts, flush=True)
