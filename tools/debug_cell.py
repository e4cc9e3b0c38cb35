import sys, torch
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs
sigma, m, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
t = inputs.config2_text(sigma); d = torch.from_numpy(t).cuda()
plans = [engine.Plan(p) for p in inputs.config2_patterns(t, sigma, m)]
obj = engine.Batch(plans) if mode == "batch" else plans
offs = torch.zeros(len(plans) + 1, dtype=torch.int64, device="cuda")
engine.find_batch_into(obj, d, None, offs); tot = int(offs[-1]); out = torch.empty(max(tot,1), dtype=torch.int64, device="cuda")
for _ in range(2): engine.find_batch_into(obj, d, out, offs)
torch.cuda.synchronize(); print("total", tot)
