"""Config-5 single pattern (a^m or a^(m-1)b) timed per launch with L2 flush (tools only)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs
m = int(sys.argv[1]); kind = sys.argv[2]; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
t = inputs.config5(); d = torch.from_numpy(t).cuda()
p = b"a" * m if kind == "am" else b"a" * (m - 1) + b"b"
pl = engine.Plan(p)
c = engine.count(pl, d)
out = torch.empty(max(c, 1), dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); engine.find_into(pl, d, out, cnt); e1.record(); torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1), 4))
gb = (t.size + 8 * c) / 1e9
print(m, kind, pl.info().family, c, ts, "GB/s(alg)=%.0f" % (gb / (min(ts) * 1e-3)), flush=True)
