"""One config-2 cell (sigma, m, anchor words, family) as a prepared batch: for ncu captures."""
import sys, torch
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs
sigma, m, nw = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fam = sys.argv[4] if len(sys.argv) > 4 else "auto"
t = inputs.config2_text(sigma); d = torch.from_numpy(t).cuda()
b = engine.Batch([engine.Plan(p, fam, anchor_words=nw) for p in inputs.config2_patterns(t, sigma, m)])
offs = torch.zeros(501, dtype=torch.int64, device="cuda")
engine.find_batch_into(b, d, None, offs); out = torch.empty(max(int(offs[-1]), 1), dtype=torch.int64, device="cuda")
for _ in range(3): engine.find_batch_into(b, d, out, offs)
torch.cuda.synchronize(); print("matches", int(offs[-1]))
