"""GPU parity against the reference's own results (tests/golden/*.json).

These compare the engine directly with digests computed by the reference
package (no oracle in between): the 10,005-case run_differential(seed=2026)
workload of the acceptance test (pkg/tests/test_acceptance.py:44-54), the
conftest fuzz sets, config 1 in full, sampled config-2 cells and 4 MiB
prefixes of configs 3-5.  Batched mode is checked on the same cases.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from cases import fuzz_cases, make_diff_case
from paper_1012_2547_b200 import engine, inputs, registry
from paper_1012_2547_b200.inputs import derive_seed

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def digest(pos) -> str:
    return hashlib.sha1(np.asarray(pos, dtype="<i8").tobytes()).hexdigest()[:16]


def test_differential_10000_seed2026(cuda):
    """Acceptance criterion 1: >= 10,000 differential cases, zero mismatches --
    every case through the descriptor of the algorithm it was drawn for."""
    fx = load("differential.json")
    mismatches, total = [], 0
    for aid, row in fx["algos"].items():
        desc = registry.get_algorithm(aid)
        for i, (sigma, n, m, kind, cnt, dg) in enumerate(row["cases"]):
            cs = derive_seed(fx["seed"], aid, i)
            _, _, _, _, p, t = make_diff_case(row["m_min"], row["m_max"], cs)
            got = desc.search(p, t)
            total += 1
            if (len(got), digest(got)) != (cnt, dg):
                mismatches.append((aid, i, sigma, n, m, kind))
    assert total >= 10000
    assert not mismatches, mismatches[:10]


@pytest.mark.parametrize("idx", range(5))
def test_fuzz_golden(cuda, idx):
    fx = load("fuzz.json")[idx]
    prm = fx["params"]
    kw = {k: v for k, v in prm.items() if k not in ("seed", "count", "m_lo", "m_hi")}
    if "sigmas" in kw:
        kw["sigmas"] = tuple(kw["sigmas"])
    for (p, t), (m, n, cd, cnt, dg) in zip(fuzz_cases(prm["seed"], prm["count"], prm["m_lo"], prm["m_hi"], **kw),
                                           fx["cases"]):
        got = engine.find(engine.Plan(p), t).cpu().numpy() if m <= n else np.empty(0, np.int64)
        assert (got.size, digest(got)) == (cnt, dg), (m, n)


def test_config1_golden(cuda):
    fx = load("configs.json")["cfg1"]
    t, pats = inputs.config1()
    got = engine.find(engine.Plan(pats[0]), t).cpu().tolist()
    assert got == fx["positions"]


def test_config2_golden_cells_batched(cuda):
    """Sampled (sigma, m) cells of config 2; each sigma's patterns go through one batched launch."""
    fx = load("configs.json")["cfg2"]
    by_sigma = {}
    for sigma, m, i, cnt, dg in fx:
        if m:
            by_sigma.setdefault(sigma, []).append((m, i, cnt, dg))
    for sigma, rows in by_sigma.items():
        t = inputs.config2_text(sigma)
        d = torch.from_numpy(t).cuda()
        pats = [t[i : i + m].tobytes() for m, i, _, _ in rows]
        pos, offs = engine.find_batch([engine.Plan(p) for p in pats], d)
        pos = pos.cpu().numpy()
        for k, (m, i, cnt, dg) in enumerate(rows):
            got = pos[offs[k] : offs[k + 1]]
            assert (got.size, digest(got)) == (cnt, dg), (sigma, m)
            single = engine.find(engine.Plan(pats[k]), d).cpu().numpy()
            assert np.array_equal(single, got)


def test_config345_golden_prefixes(cuda):
    fx = load("configs.json")
    t3 = inputs.zipf_text(4 << 20, derive_seed(inputs.ROOT_SEED, "cfg3", "text"))
    d3 = torch.from_numpy(t3).cuda()
    for m, i, cnt, dg in fx["cfg3_4MiB"]["rows"]:
        got = engine.find(engine.Plan(t3[i : i + m].tobytes()), d3).cpu().numpy()
        assert (got.size, digest(got)) == (cnt, dg), ("cfg3", m)
    t4 = inputs.config4_text(4 << 20)
    d4 = torch.from_numpy(t4).cuda()
    for m, i, cnt, dg in fx["cfg4_4MiB"]["rows"]:
        got = engine.find(engine.Plan(t4[i : i + m].tobytes()), d4).cpu().numpy()
        assert (got.size, digest(got)) == (cnt, dg), ("cfg4", m)
    t5 = inputs.dense_text(4 << 20, derive_seed(inputs.ROOT_SEED, "cfg5", "text"))
    d5 = torch.from_numpy(t5).cuda()
    for ph, cnt, dg in fx["cfg5_4MiB"]["rows"]:
        got = engine.find(engine.Plan(bytes.fromhex(ph)), d5).cpu().numpy()
        assert (got.size, digest(got)) == (cnt, dg), ("cfg5", len(ph) // 2)
