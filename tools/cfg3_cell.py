"""One config-3 batch (m) timed with L2 flush per rep; prints per-rep ms (tools only)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs
m = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t = inputs.config3(); d = torch.from_numpy(t).cuda()
b = engine.Batch([engine.Plan(p) for p in inputs.config3_patterns(t, m)])
offs = torch.zeros(501, dtype=torch.int64, device="cuda")
engine.find_batch_into(b, d, None, offs); out = torch.empty(max(int(offs[-1]), 1), dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mp0 = engine.mp_batches()
ts = []
for _ in range(reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); engine.find_batch_into(b, d, out, offs); e1.record(); torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1), 4))
print(m, "mp", engine.mp_batches() - mp0, ts, flush=True)
