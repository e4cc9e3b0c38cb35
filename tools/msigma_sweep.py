"""Single-pattern roofline sweep over sigma x m on a >= 1 GiB HBM-resident text
(PAPER.md's Rand-sigma grid at B200 scale).

For each sigma in {2, 4, 16, 64, 256}: a 1 GiB i.i.d. uniform text (generated
on the device, seeded), and for each m in DEFAULT_LENGTHS + {3, 5, 6, 7, 12}
one pattern copied from a random text offset.  Each search is timed with CUDA
events on the launching stream (median of 5 after 2 warm-ups; the text is 8x
L2, no flush needed) and emits every position.  Algorithmic bytes per search
B = n + 8*count + 8; frac_8tbs = B/t / 8e12 (the north
star's ~8 TB/s), frac_copy = B/t / MEASURED_PEAKS hbm_gbs.  Counts are checked
against the threaded C oracle for a spread of cells (--check).

usage: python tools/msigma_sweep.py [--gib 1] [--check] > profiles/r2/msigma_sweep.jsonl
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import measured_peak  # noqa: E402
from paper_1012_2547_b200 import engine  # noqa: E402
from paper_1012_2547_b200.inputs import DEFAULT_LENGTHS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=1.0)
ap.add_argument("--check", action="store_true")
ap.add_argument("--sigmas", default="2,4,16,64,256")
ap.add_argument("--lengths", default="")
ap.add_argument("--family", default="auto")
ap.add_argument("--no-hist", action="store_true", help="plan without the text's byte histogram (K0)")
args = ap.parse_args()

n = int(args.gib * (1 << 30))
peak, _ = measured_peak()
lengths = sorted(set(DEFAULT_LENGTHS) | {3, 5, 6, 7, 12}) if not args.lengths else [int(x) for x in args.lengths.split(",")]
out = torch.empty(n // 4 + (1 << 20), dtype=torch.int64, device="cuda")  # sigma = 2, m = 2: n/4 positions
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for sigma in [int(x) for x in args.sigmas.split(",")]:
    g = torch.Generator(device="cuda").manual_seed(2026 + sigma)
    d = torch.randint(0, sigma, (n,), dtype=torch.uint8, device="cuda", generator=g)
    h = d.cpu().numpy() if args.check else None
    rng = np.random.default_rng(sigma)
    # the text's byte histogram (K0 on the device) goes to the planner, as the reference's
    # select(pattern, text) sees the text's alphabet (registry.py:209-222)
    hist = None if args.no_hist else engine.histogram(d).cpu().numpy()
    for m in lengths:
        off = int(rng.integers(0, n - m))
        p = d[off : off + m].cpu().numpy().tobytes()
        try:
            pl = engine.Plan(p, args.family, hist=hist)
        except ValueError:
            continue
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
        B = n + 8 * c + 8
        rate = B / (ms * 1e-3) / 1e9
        row = {"sigma": sigma, "m": m, "family": inf.family, "words": inf.words, "count": c, "ms": round(ms, 4),
               "text_gbps": round(n / (ms * 1e-3) / 1e9, 1), "alg_gbps": round(rate, 1),
               "frac_8tbs": round(rate / 8000.0, 3), "frac_copy": round(rate / peak, 3)}
        if args.check and (m in (2, 8, 64, 1024) or sigma in (2, 256)):
            import oracle

            want = oracle.count(p, h, threads=os.cpu_count() or 4)
            row["oracle_count_ok"] = bool(want == c)
            if c <= out.numel() and c <= (1 << 22):
                got = out[:c].cpu().numpy()
                row["positions_ok"] = bool(np.array_equal(got, oracle.search(p, h, threads=os.cpu_count() or 4)))
        print(json.dumps(row), flush=True)
    del d
