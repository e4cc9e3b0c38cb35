"""Single-pattern throughput across m on a sigma=256 text (default 4 GiB, HBM-resident,
larger than L2): median of 5 event-timed searches per m; writes one JSON line per m.
usage: m_sweep.py [GiB] (tools only)"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from bench import measured_peak  # noqa: E402
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gib * (1 << 30))
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
inputs.config4_text(n, out=host.numpy())
d = host.cuda()
t = host.numpy()
peak, _ = measured_peak()
out = torch.empty(1 << 22, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for m in (2, 3, 4, 5, 6, 7, 8, 12, 16, 32, 64, 128, 200, 271, 272, 300, 400, 512, 768, 1024):
    off = (n // 3) + 17 * m
    pl = engine.Plan(t[off:off + m].tobytes())
    for _ in range(2):
        engine.find_into(pl, d, out, cnt)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.find_into(pl, d, out, cnt)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    c = int(cnt.item())
    inf = pl.info()
    gbs = n / (ms * 1e-3) / 1e9
    print(json.dumps({"m": m, "family": inf.family, "count": c, "ms": round(ms, 4), "text_gbps": round(gbs, 1),
                      "frac_of_copy_peak": round((n + 8 * c) / (ms * 1e-3) / 1e9 / peak, 3)}), flush=True)
