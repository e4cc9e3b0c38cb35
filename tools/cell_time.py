"""One config-2 cell as a prepared batch, L2-flushed median of 7 launches (tools only).
usage: cell_time.py SIGMA M"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from bench import L2Flush  # noqa: E402
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

sigma, m = int(sys.argv[1]), int(sys.argv[2])
t = inputs.config2_text(sigma)
d = torch.from_numpy(t).cuda()
b = engine.Batch([engine.Plan(p) for p in inputs.config2_patterns(t, sigma, m)])
offs = torch.zeros(len(b) + 1, dtype=torch.int64, device="cuda")
engine.find_batch_into(b, d, None, offs)
out = torch.empty(max(int(offs[-1]), 1), dtype=torch.int64, device="cuda")
flush = L2Flush(torch.device("cuda"))
ts = []
for _ in range(7):
    flush()
    torch.cuda._sleep(400_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    engine.find_batch_into(b, d, out, offs)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{statistics.median(ts):.4f} ms  matches {int(offs[-1])}")
