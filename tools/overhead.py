"""Per-search fixed cost: host enqueue time and GPU time for small texts (tools only)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs
for n in (1 << 10, 1 << 20, 64 << 20):
    t = inputs.rand_text_np(256, n, 5)
    d = torch.from_numpy(t).cuda()
    pl = engine.Plan(t[100:108].tobytes())
    out = torch.empty(1 << 16, dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(20): engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
    N = 200
    t0 = time.perf_counter()
    for _ in range(N): engine.find_into(pl, d, out, cnt)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N): engine.find_into(pl, d, out, cnt)
    e1.record(); torch.cuda.synchronize()
    print(f"n={n:>10} enqueue {1e6*(t1-t0)/N:7.1f} us/call  drain {1e6*(t2-t0)/N:7.1f} us/call  events {1e3*e0.elapsed_time(e1)/N:7.1f} us/call", flush=True)
x = torch.empty(1, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(1000): x.add_(1)
torch.cuda.synchronize(); print(f"torch add_ launch: {1e6*(time.perf_counter()-t0)/1000:.1f} us/call")
