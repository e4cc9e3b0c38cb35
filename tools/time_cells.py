import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs
for sigma, m in ((2, 64), (128, 2), (16, 16)):
    t = inputs.config2_text(sigma); d = torch.from_numpy(t).cuda()
    pats = inputs.config2_patterns(t, sigma, m)
    plans = [engine.Plan(p) for p in pats]
    for mode in ("list", "batch"):
        obj = engine.Batch(plans) if mode == "batch" else plans
        offs = torch.zeros(len(plans) + 1, dtype=torch.int64, device="cuda")
        engine.find_batch_into(obj, d, None, offs); tot = int(offs[-1]); out = torch.empty(max(tot,1), dtype=torch.int64, device="cuda")
        for _ in range(3): engine.find_batch_into(obj, d, out, offs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        for _ in range(5): engine.find_batch_into(obj, d, out, offs)
        e1.record(); torch.cuda.synchronize()
        print(sigma, m, mode, "events %.3f ms" % (e0.elapsed_time(e1) / 5), "wall %.3f ms" % ((time.perf_counter() - t0) * 200), flush=True)
