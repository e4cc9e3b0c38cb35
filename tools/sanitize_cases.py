"""Small searches over every kernel family and edge case, for
`compute-sanitizer --tool memcheck` (tools only; exits non-zero on a mismatch)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1012_2547_b200 import engine, search_many  # noqa: E402

TILE = 16384
rng = np.random.default_rng(1)


def check(p, t, family="auto", off=0):
    base = torch.from_numpy(np.frombuffer(t + b"\0" * 32, dtype=np.uint8).copy()).cuda()
    view = base[off : len(t)]
    got = engine.find(engine.Plan(p, family), view).cpu().numpy()
    want = oracle.search(p, t[off:])
    assert np.array_equal(got, want), (len(p), family, off)


def rb(sigma, n):
    return rng.integers(0, sigma, n, dtype=np.uint8).tobytes()


n = 2 * TILE + 1234
for sigma in (2, 4, 256):
    t = rb(sigma, n)
    for m in (1, 2, 3, 4, 5, 7, 16, 33, 64, 65, 300, 1024, 3000):
        if m > n:
            continue
        i = int(rng.integers(0, n - m))
        p = t[i : i + m]
        for off in (0, 5):
            check(p, t, "auto", off)
        if m >= 4:
            check(p, t, "win4")
        if m >= 7:
            check(p, t, "aligned")
        if m <= 64:
            check(p, t, "shiftor")
        if m >= 15:
            check(p, t, "gram")
            check(p, t, "gram", 5)
dense = bytearray(b"a" * n)
for i in rng.choice(n, 40, replace=False):
    dense[i] = ord("b")
dense = bytes(dense)
for m in (2, 16, 128, 1024):
    check(b"a" * m, dense)
    check(b"a" * (m - 1) + b"b", dense)
t = rb(256, 4 * TILE)
pats = [t[i : i + 24] for i in rng.integers(0, 4 * TILE - 24, 40)] + [rb(256, 9)]
res = search_many(pats, t)
for p, r in zip(pats, res):
    assert r == oracle.search(p, t).tolist()
# batched passes: K5 (aligned words), K5b (byte offsets, q = 2 / 4 / 8 / 16) with
# dense patterns left to their scans, anchor words 2 / 3, sampled in a batch,
# duplicate patterns
for sigma, lo, hi in ((256, 8, 40), (16, 2, 3), (64, 4, 6), (4, 8, 30), (32, 300, 1200), (2, 16, 300)):
    t = rb(sigma, 3 * TILE + 321)
    ms = rng.integers(lo, hi + 1, 64)
    pats = [t[i : i + m] for i, m in zip(rng.integers(0, len(t) - hi, 64), ms)] + [b"ab" * 2, t[:lo]]
    pats += pats[:5]
    for obj in (None, "prepared"):
        plans = [engine.Plan(p) for p in pats]
        pos, offs = engine.find_batch(engine.Batch(plans) if obj else plans, t)
        pos = pos.cpu().numpy()
        for k, p in enumerate(pats):
            assert np.array_equal(pos[offs[k] : offs[k + 1]], oracle.search(p, t)), (sigma, k)
for nw in (2, 3):
    t = rb(2, 2 * TILE + 77)
    p = t[1000:1040]
    got = engine.find(engine.Plan(p, anchor_words=nw), t).cpu().numpy()
    assert np.array_equal(got, oracle.search(p, t)), nw
torch.cuda.synchronize()
print("sanitize cases ok")
