"""Per-kernel device times of a few searches via torch.profiler (CUPTI activity
records: real clocks, no replay).  usage: kprof.py cfg5 <m> <am|amb> | cfg2 <sigma> <m> (tools only)."""
import sys, torch
sys.path.insert(0, '.')
from torch.profiler import profile, ProfilerActivity
from paper_1012_2547_b200 import engine, inputs

mode = sys.argv[1]
if mode == "cfg5":
    m, kind = int(sys.argv[2]), sys.argv[3]
    t = inputs.config5(); d = torch.from_numpy(t).cuda()
    pl = engine.Plan(b"a" * m if kind == "am" else b"a" * (m - 1) + b"b")
    c = engine.count(pl, d)
    out = torch.empty(max(c, 1), dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    run = lambda: engine.find_into(pl, d, out, cnt)
elif mode == "rand":  # rand <MiB> <m> <family>
    n, m, fam = int(sys.argv[2]) << 20, int(sys.argv[3]), sys.argv[4]
    t = inputs.rand_text_np(256, n, 11); d = torch.from_numpy(t).cuda()
    pl = engine.Plan(t[n // 2 : n // 2 + m].tobytes(), fam)
    c = engine.count(pl, d)
    out = torch.empty(max(c, 1), dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    run = lambda: engine.find_into(pl, d, out, cnt)
else:
    sigma, m = int(sys.argv[2]), int(sys.argv[3])
    t = inputs.config2_text(sigma) if sigma != 95 else inputs.config3()
    d = torch.from_numpy(t).cuda()
    pats = inputs.config2_patterns(t, sigma, m) if sigma != 95 else inputs.config3_patterns(t, m)
    b = engine.Batch([engine.Plan(p) for p in pats])
    offs = torch.zeros(501, dtype=torch.int64, device="cuda")
    engine.find_batch_into(b, d, None, offs); out = torch.empty(max(int(offs[-1]), 1), dtype=torch.int64, device="cuda")
    run = lambda: engine.find_batch_into(b, d, out, offs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3): run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        flush.zero_()
        run()
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA" and "mb::" in e.name:
        k = e.name.split("(")[0][-40:]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:<42} n={n:>3} avg={us / n:9.1f} us")
