"""A few single-pattern searches over one text size (for ncu launch lists; tools only).
usage: small_search.py N_BYTES [SIGMA] [M] [REPS]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

n = int(sys.argv[1])
sigma = int(sys.argv[2]) if len(sys.argv) > 2 else 256
m = int(sys.argv[3]) if len(sys.argv) > 3 else 16
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
t = inputs.rand_text_np(sigma, n, 3)
d = torch.from_numpy(t).cuda()
pl = engine.Plan(t[n // 3:n // 3 + m].tobytes())
out = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(reps):
    engine.find_into(pl, d, out, cnt)
torch.cuda.synchronize()
print("count", int(cnt.item()), "family", pl.info().family)
