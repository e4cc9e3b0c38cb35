"""GPU parity at the BASELINE.json configs' full sizes.

Exact parity against the C oracle (oracle/, threaded over halo-overlapped
chunks -- SURVEY.md 8(c)) plus size-independent properties: positions strictly
increasing, every reported window equal to the pattern (host check), planted
occurrences present, batched == single-pattern results.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1012_2547_b200 import engine, inputs
from paper_1012_2547_b200.inputs import derive_seed

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = os.cpu_count() or 4


def props(pos: np.ndarray, p: bytes, t: np.ndarray):
    assert pos.dtype == np.int64
    if pos.size:
        assert np.all(np.diff(pos) > 0), "positions not strictly increasing"
        assert pos[0] >= 0 and pos[-1] <= t.size - len(p)
        pv = np.frombuffer(p, dtype=np.uint8)
        sample = pos if pos.size <= 4096 else pos[np.linspace(0, pos.size - 1, 4096).astype(np.int64)]
        win = t[sample[:, None] + np.arange(len(p))[None, :]]
        assert np.all(win == pv[None, :]), "a reported window differs from the pattern"


def test_config1_full(cuda):
    t, pats = inputs.config1()
    got = engine.find(engine.Plan(pats[0]), t).cpu().numpy()
    assert np.array_equal(got, oracle.search(pats[0], t))
    props(got, pats[0], t)


def _digests():
    with open(os.path.join(os.path.dirname(__file__), "golden", "cfg23_digests.json")) as f:
        return json.load(f)


def digest(pos: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(pos, dtype="<i8").tobytes()).hexdigest()[:16]


def check_every_list(pos: np.ndarray, offs: np.ndarray, want: list, tag) -> None:
    """Every pattern's CSR slice: count and digest of all positions
    (tests/golden/make_cfg23_digests.py, C oracle brute force)."""
    assert offs.size == len(want) + 1 and offs[0] == 0
    bad = []
    for k, (cnt, dg) in enumerate(want):
        got = pos[offs[k] : offs[k + 1]]
        if got.size != cnt or digest(got) != dg:
            bad.append((k, got.size, cnt))
    assert not bad, (tag, f"{len(bad)} of {len(want)} lists differ", bad[:5])


@pytest.mark.parametrize("sigma", [2, 4, 8, 16, 32, 64, 128])
def test_config2_full_sigma(cuda, sigma):
    """All 10 m x 500 patterns of one sigma: one batched launch per m; EVERY
    pattern's full position list against its oracle digest; single-pattern
    searches for a spread of patterns."""
    gold = _digests()
    t = inputs.config2_text(sigma)
    assert hashlib.sha1(t.tobytes()).hexdigest()[:16] == gold["texts"][f"cfg2_{sigma}"], "text generator drifted"
    d = torch.from_numpy(t).cuda()
    for m in inputs.DEFAULT_LENGTHS:
        pats = inputs.config2_patterns(t, sigma, m)
        want = gold["cfg2"][str(sigma)][str(m)]
        batch = engine.Batch([engine.Plan(p) for p in pats])
        pos, offs = engine.find_batch(batch, d)
        pos = pos.cpu().numpy()
        offs = offs.numpy()
        check_every_list(pos, offs, want, (sigma, m, "batched"))
        for k in range(0, len(pats), 50):
            props(pos[offs[k] : offs[k + 1]], pats[k], t)
        for k in range(3, len(pats), 61):  # single-pattern path on a spread
            got = engine.find(engine.Plan(pats[k]), d).cpu().numpy()
            assert got.size == want[k][0] and digest(got) == want[k][1], (sigma, m, k, "single")


def test_config3_full(cuda):
    gold = _digests()
    t = inputs.config3()
    assert hashlib.sha1(t.tobytes()).hexdigest()[:16] == gold["texts"]["cfg3"], "text generator drifted"
    d = torch.from_numpy(t).cuda()
    for m in (4, 16, 64, 256, 1024):
        pats = inputs.config3_patterns(t, m)
        want = gold["cfg3"][str(m)]
        before = engine.mp_batches()
        pos, offs = engine.find_batch([engine.Plan(p) for p in pats], d)
        if m in (16, 64, 256, 1024):
            assert engine.mp_batches() == before + 1, f"cfg3 m={m} batch did not take the MP pass"
        pos = pos.cpu().numpy()
        offs = offs.numpy()
        check_every_list(pos, offs, want, (m, "batched"))
        props(pos[offs[0] : offs[1]], pats[0], t)
        for k in range(7, len(pats), 49):
            got = engine.find(engine.Plan(pats[k]), d).cpu().numpy()
            assert got.size == want[k][0] and digest(got) == want[k][1], (m, k, "single")


def test_config5_full(cuda):
    t = inputs.config5()
    d = torch.from_numpy(t).cuda()
    for p in inputs.config5_patterns():
        got = engine.find(engine.Plan(p), d).cpu().numpy()
        want = oracle.search(p, t, "SO", threads=THREADS)  # BF is O(n*m) on a^m
        assert np.array_equal(got, want), (len(p), p[-1:], got.size, want.size,
                                           sorted(set(want.tolist()) - set(got.tolist()))[:5],
                                           sorted(set(got.tolist()) - set(want.tolist()))[:5])
        props(got, p, t)


def test_config4_full(cuda):
    n = 16 << 30
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t = host.numpy()
    inputs.config4_text(n, out=t)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(host)
    for p in inputs.config4_patterns(t):
        got = engine.find(engine.Plan(p), d).cpu().numpy()
        assert np.array_equal(got, oracle.search(p, t, threads=THREADS)), len(p)
        props(got, p, t)
    del d
    torch.cuda.empty_cache()


def test_large_text_batch_keeps_the_pass_per_sub_batch(cuda, monkeypatch):
    """A 256 MiB text against 96 patterns with a scratch budget that fits ~40
    patterns: the batch runs as 3 chained sub-batches, each planned on its own
    and each still ONE pass over the text (not one scan per pattern); every
    position of every pattern equals the threaded C oracle."""
    n = 256 << 20
    t = inputs.rand_text_np(64, n, derive_seed(2026, "large-batch"))
    rng = np.random.default_rng(77)
    pats = []
    for i in range(96):
        m = int(rng.integers(12, 41))
        off = int(rng.integers(0, n - m))
        pats.append(t[off : off + m].tobytes())
    pats[17] = pats[3]  # a duplicate inside one sub-batch
    pats[70] = pats[5]  # ... and one whose first copy sits in an earlier sub-batch
    d = torch.from_numpy(t).cuda()
    plans = engine.Batch([engine.Plan(p) for p in pats])
    per_pattern = (n // 2048 + 64) * 346
    monkeypatch.setenv("MB_SCRATCH_BUDGET", str(per_pattern * 40))
    before = engine.mp_batches()
    pos, offs = engine.find_batch(plans, d)
    assert engine.mp_batches() == before + 3, "a sub-batch fell back to per-pattern scans"
    pos, offs = pos.cpu().numpy(), offs.cpu().numpy()
    assert offs[0] == 0 and offs.size == len(pats) + 1
    for k, p in enumerate(pats):
        want = oracle.search(p, t, threads=THREADS)
        assert np.array_equal(pos[offs[k] : offs[k + 1]], want), k
    # the ad-hoc entry (mb_find_batch: plans given per call) takes the same route
    before = engine.mp_batches()
    pos2, offs2 = engine.find_batch([engine.Plan(p) for p in pats], d)
    assert engine.mp_batches() == before + 3
    assert np.array_equal(pos2.cpu().numpy(), pos) and np.array_equal(offs2.cpu().numpy(), offs)
