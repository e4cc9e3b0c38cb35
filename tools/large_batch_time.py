"""Batched search of one large text (default 1 GiB, Zipf-like printable bytes as
config 3) against 500 patterns, event-timed: the batch runs as sub-batches under
the scratch budget, each still one pass over the text (tools only).
usage: python tools/large_batch_time.py [GiB] [m]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker of a sample of the lists)
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
m = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n = int(gib * (1 << 30))
base = inputs.config3()  # 64 MiB
t = np.tile(base, (n + base.size - 1) // base.size)[:n]
rng = np.random.default_rng(5)
pats = [t[o : o + m].tobytes() for o in rng.integers(0, n - m, 500)]
d = torch.from_numpy(t).cuda()
b = engine.Batch([engine.Plan(p) for p in pats])
offs = torch.zeros(501, dtype=torch.int64, device="cuda")
engine.find_batch_into(b, d, None, offs)
total = int(offs[-1])
out = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
mp0, l0 = engine.mp_batches(), engine.launch_count()
engine.find_batch_into(b, d, out, offs)
torch.cuda.synchronize()
passes, launches = engine.mp_batches() - mp0, engine.launch_count() - l0
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    engine.find_batch_into(b, d, out, offs)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
o = offs.cpu().numpy()
pos = out.cpu().numpy()
bad = 0
for k in range(0, 500, 50):
    bad += not np.array_equal(pos[o[k] : o[k + 1]], oracle.search(pats[k], t, threads=os.cpu_count() or 4))
print(f"{gib} GiB x 500 patterns (m={m}): {min(ts):.3f} ms, {passes} passes, {launches} launches, "
      f"{total} matches, aggregated {500 * n / (min(ts) * 1e-3) / 1e12:.1f} TB/s, sampled lists wrong: {bad}")
