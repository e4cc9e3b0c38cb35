"""Kernel-phase timeline of the config-5 sparse searches (trace build; tools only)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs
NAMES = {0: "scan entry", 1: "scan exit (last)", 2: "offsets entry", 4: "offsets after wait (first)", 5: "offsets after wait (last)", 24: "published (first)", 25: "published (last)", 7: "prefix done (last)", 9: "offsets exit (last)", 10: "expand entry", 12: "expand after wait", 13: "expand exit"}
L = engine.load_library(); L.mb_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
t = inputs.config5(); d = torch.from_numpy(t).cuda()
for p in (b"ab", b"a" * 15 + b"b"):
    pl = engine.Plan(p); out = torch.empty(1 << 20, dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    buf = np.zeros(32, dtype=np.uint64)
    for rep in range(4):
        torch.cuda.synchronize(); L.mb_debug_trace(None, 1); torch.cuda._sleep(1_000_000)
        engine.find_into(pl, d, out, cnt); torch.cuda.synchronize(); L.mb_debug_trace(buf.ctypes.data, 0)
    t0 = int(buf[0]); print(p[-2:], "count", int(cnt.item()))
    for i in sorted(NAMES, key=lambda i: int(buf[i])):
        v = int(buf[i])
        if v not in (0, 2**64 - 1): print(f"  {(v - t0) / 1e3:8.2f} us  {NAMES[i]}")
