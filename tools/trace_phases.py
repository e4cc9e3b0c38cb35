"""Kernel-phase timeline of one search (trace build, %globaltimer marks; tools only).
usage: MB_ENGINE_LIB=paper_1012_2547_b200/libmatchb200_trace.so python tools/trace_phases.py N [SIGMA] [M]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

NAMES = {0: "scan entry (first CTA)", 1: "scan exit (last CTA)", 2: "offsets entry (first)",
         4: "offsets after pdl_wait (first)", 5: "offsets after pdl_wait (last)", 7: "offsets after look-back (last)",
         9: "offsets exit (last)", 10: "expand entry (first)", 12: "expand after pdl_wait (first)",
         13: "expand exit (last)", 14: "fused: scan done (first)", 15: "fused: scan done (last)",
         16: "fused: barrier 1 passed (first)", 17: "fused: barrier 1 passed (last)",
         19: "fused: offsets done (last)", 24: "offsets aggregate published (first)",
         25: "offsets aggregate published (last)", 20: "fused: barrier 2 passed (first)", 21: "fused: exit (last)"}

n = int(sys.argv[1])
sigma = int(sys.argv[2]) if len(sys.argv) > 2 else 256
m = int(sys.argv[3]) if len(sys.argv) > 3 else 16
L = engine.load_library()
L.mb_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
t = inputs.rand_text_np(sigma, n, 3)
d = torch.from_numpy(t).cuda()
pl = engine.Plan(t[n // 3:n // 3 + m].tobytes())
out = torch.empty(1 << 22, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
buf = np.zeros(32, dtype=np.uint64)
for rep in range(6):
    torch.cuda.synchronize()
    assert L.mb_debug_trace(None, 1) == 0
    torch.cuda._sleep(1_000_000)
    engine.find_into(pl, d, out, cnt)
    torch.cuda.synchronize()
    L.mb_debug_trace(buf.ctypes.data, 0)
    if rep < 3:
        continue
    t0 = int(buf[0])
    print(f"n={n} sigma={sigma} m={m} count={int(cnt.item())} family={pl.info().family}")
    for i in sorted(NAMES):
        v = int(buf[i])
        if v in (0, 2**64 - 1):
            continue
        print(f"  {(v - t0) / 1e3:8.2f} us  {NAMES[i]}")
