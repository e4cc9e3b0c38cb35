"""Kernel-phase timeline of one config-3 batch (trace build, %globaltimer marks; tools only).
usage: MB_ENGINE_LIB=paper_1012_2547_b200/libmatchb200_trace.so python tools/trace_batch.py [m]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

NAMES = {0: "gated scan entry (first CTA)", 1: "gated scan exit (last CTA)", 2: "offsets entry (first)",
         4: "offsets after pdl_wait (first)", 5: "offsets after pdl_wait (last)", 24: "offsets aggregate published (first)",
         25: "offsets aggregate published (last)", 7: "offsets after look-back (last)",
         9: "offsets exit (last)", 10: "expand entry (first)", 12: "expand after pdl_wait (first)",
         13: "expand exit (last)"}
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
L = engine.load_library()
L.mb_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
t = inputs.config3()
d = torch.from_numpy(t).cuda()
b = engine.Batch([engine.Plan(p) for p in inputs.config3_patterns(t, m)])
offs = torch.zeros(501, dtype=torch.int64, device="cuda")
out = torch.empty(1 << 22, dtype=torch.int64, device="cuda")
buf = np.zeros(32, dtype=np.uint64)
for rep in range(6):
    torch.cuda.synchronize()
    assert L.mb_debug_trace(None, 1) == 0
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    engine.find_batch_into(b, d, out, offs)
    e1.record()
    torch.cuda.synchronize()
    L.mb_debug_trace(buf.ctypes.data, 0)
    if rep < 3:
        continue
    t0 = int(buf[2])
    print(f"cfg3 m={m}: batch {e0.elapsed_time(e1) * 1e3:.1f} us; times relative to offsets entry")
    for i in sorted(NAMES, key=lambda i: int(buf[i])):
        v = int(buf[i])
        if v in (0, 2**64 - 1):
            continue
        print(f"  {(v - t0) / 1e3:8.2f} us  {NAMES[i]}")
