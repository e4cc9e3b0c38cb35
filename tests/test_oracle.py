"""CPU: pin the oracle restatement (oracle/oracle.c) to the reference.

Every expectation comes from tests/golden/*.json, produced by running the
reference itself (tests/golden/make_golden.py).  The case generators used here
(tests/cases.py, paper_1012_2547_b200/inputs.py) are pinned too: a digest of
each generated case / text is part of the fixture.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from cases import KNOWN, fuzz_cases, make_diff_case
from paper_1012_2547_b200 import inputs
from paper_1012_2547_b200.inputs import derive_seed

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def digest(pos) -> str:
    return hashlib.sha1(np.asarray(pos, dtype="<i8").tobytes()).hexdigest()[:16]


def tdigest(b: bytes) -> str:
    return hashlib.sha1(b).hexdigest()[:16]


ALL = list(oracle.ALGOS)


def test_known_answers_all_algorithms():
    for p, t, exp in KNOWN:
        for a in ALL:
            try:
                got = oracle.search(p, t, a).tolist()
            except ValueError:
                continue  # outside the algorithm's bounds
            assert got == exp, (a, p[:8], t[:8])


@pytest.mark.parametrize("idx", range(5))
def test_fuzz_golden(idx):
    fx = load("fuzz.json")[idx]
    prm = fx["params"]
    kw = {k: v for k, v in prm.items() if k not in ("seed", "count", "m_lo", "m_hi")}
    if "sigmas" in kw:
        kw["sigmas"] = tuple(kw["sigmas"])
    cases = list(fuzz_cases(prm["seed"], prm["count"], prm["m_lo"], prm["m_hi"], **kw))
    assert len(cases) == len(fx["cases"])
    for (p, t), (m, n, cd, cnt, dg) in zip(cases, fx["cases"]):
        assert (len(p), len(t), tdigest(p + b"|" + t)) == (m, n, cd), "case generator drifted"
        r = oracle.search(p, t)
        assert (r.size, digest(r)) == (cnt, dg)
        assert r.tolist() == oracle.naive_scan(p, t)


def test_differential_golden_subset():
    """run_differential(seed=2026) cases (differential.py:70-131) -- 40 per algorithm on CPU."""
    fx = load("differential.json")
    for aid, row in fx["algos"].items():
        for i, (sigma, n, m, kind, cnt, dg) in enumerate(row["cases"][:40]):
            cs = derive_seed(fx["seed"], aid, i)
            s2, n2, m2, k2, p, t = make_diff_case(row["m_min"], row["m_max"], cs)
            assert (s2, n2, m2, k2[0]) == (sigma, n, m, kind)
            r = oracle.search(p, t, "SO" if m > 64 else "BF")
            assert (r.size, digest(r)) == (cnt, dg), (aid, i)


def test_tables_golden():
    from paper_1012_2547_b200 import engine

    for row in load("tables.json"):
        p = bytes.fromhex(row["p"])
        assert oracle.horspool_table(p) == row["hor"]
        assert oracle.sunday_table(p) == row["sun"]
        plan = engine.Plan(p)  # host-side tables (H1) of the product; no GPU needed
        assert plan.horspool_table() == row["hor"]
        assert plan.sunday_table() == row["sun"]
        assert plan.kmp_failure() == row["kmp"]
        fm = plan.forward_masks()
        want = [0] * 256
        for c, v in row["fwd"].items():
            want[int(c)] = int(v, 16)
        assert fm == want
        for q, hs in row["gram"].items():
            assert plan.gram_hashes(int(q)) == hs


def test_config1_golden():
    fx = load("configs.json")["cfg1"]
    t, pats = inputs.config1()
    assert tdigest(t.tobytes()) == fx["text"]
    assert pats[0].hex() == fx["pattern"]
    assert oracle.search(pats[0], t).tolist() == fx["positions"]


def test_config2_golden_sample():
    fx = load("configs.json")["cfg2"]
    texts = {}
    for sigma, m, i, cnt, dg in fx:
        if m == 0:
            t = texts.setdefault(sigma, inputs.config2_text(sigma))
            assert tdigest(t.tobytes()) == dg
    for sigma, m, i, cnt, dg in fx[:: 7]:
        if m == 0:
            continue
        t = texts.setdefault(sigma, inputs.config2_text(sigma))
        offs = inputs.sample_positions(t.size, m, 500, derive_seed(inputs.ROOT_SEED, "cfg2", sigma, m))
        assert i in offs[:2]
        p = t[i : i + m].tobytes()
        r = oracle.search(p, t, threads=4)
        assert (r.size, digest(r)) == (cnt, dg)


def test_config345_golden_prefixes():
    fx = load("configs.json")
    t3 = inputs.zipf_text(4 << 20, derive_seed(inputs.ROOT_SEED, "cfg3", "text"))
    assert tdigest(t3.tobytes()) == fx["cfg3_4MiB"]["text"]
    for m, i, cnt, dg in fx["cfg3_4MiB"]["rows"]:
        r = oracle.search(t3[i : i + m].tobytes(), t3, threads=4)
        assert (r.size, digest(r)) == (cnt, dg)
    t4 = inputs.config4_text(4 << 20)
    assert tdigest(t4.tobytes()) == fx["cfg4_4MiB"]["text"]
    for m, i, cnt, dg in fx["cfg4_4MiB"]["rows"]:
        r = oracle.search(t4[i : i + m].tobytes(), t4, threads=4)
        assert (r.size, digest(r)) == (cnt, dg)
    t5 = inputs.dense_text(4 << 20, derive_seed(inputs.ROOT_SEED, "cfg5", "text"))
    assert tdigest(t5.tobytes()) == fx["cfg5_4MiB"]["text"]
    for ph, cnt, dg in fx["cfg5_4MiB"]["rows"]:
        r = oracle.search(bytes.fromhex(ph), t5, "SO", threads=4)
        assert (r.size, digest(r)) == (cnt, dg)


def test_threaded_chunking_matches_single():
    rng = np.random.default_rng(3)
    for _ in range(200):
        sigma = int(rng.choice([1, 2, 4, 256]))
        n = int(rng.integers(0, 3000))
        m = int(rng.integers(1, 40))
        t = rng.integers(0, sigma, n, dtype=np.uint8).tobytes()
        p = rng.integers(0, sigma, m, dtype=np.uint8).tobytes()
        k = int(rng.integers(2, 17))
        assert oracle.search(p, t, threads=k).tolist() == oracle.search(p, t).tolist()


# The algorithms the CPU legs of bench.py time (the reference's auto path on
# configs 3-5: FJS, EBOM, SSEF, LBNDM -- registry.py:209-222) and the other
# restated searchers, each against the reference-generated digests of every
# fuzz and differential case inside its applicability bounds.
BOUNDS = {"SSEF": (32, None), "EBOM": (2, None), "FSBNDM": (1, 63), "HASH3": (3, None), "HASH5": (5, None),
          "HASH8": (8, None)}


@pytest.mark.parametrize("algo", [a for a in ALL if a != "BF"])
def test_fuzz_and_differential_golden_per_algorithm(algo):
    lo, hi = BOUNDS.get(algo, (1, None))
    ran = 0
    for fx in load("fuzz.json"):
        prm = fx["params"]
        kw = {k: v for k, v in prm.items() if k not in ("seed", "count", "m_lo", "m_hi")}
        if "sigmas" in kw:
            kw["sigmas"] = tuple(kw["sigmas"])
        for (p, t), (m, n, cd, cnt, dg) in zip(fuzz_cases(prm["seed"], prm["count"], prm["m_lo"], prm["m_hi"], **kw),
                                                fx["cases"]):
            if m < lo or (hi is not None and m > hi):
                continue
            r = oracle.search(p, t, algo)
            assert (r.size, digest(r)) == (cnt, dg), (algo, "fuzz", prm["seed"], m, n)
            ran += 1
    fx = load("differential.json")
    for aid, row in fx["algos"].items():
        for i, (sigma, n, m, kind, cnt, dg) in enumerate(row["cases"][::4]):
            if m < lo or (hi is not None and m > hi) or (m > 256 and algo in ("HOR", "QS", "BR", "TVSBS", "BOM")):
                continue
            _, _, _, _, p, t = make_diff_case(row["m_min"], row["m_max"], derive_seed(fx["seed"], aid, 4 * i))
            r = oracle.search(p, t, algo)
            assert (r.size, digest(r)) == (cnt, dg), (algo, "differential", aid, 4 * i)
            ran += 1
    assert ran >= 500, ran


def test_cfg23_digests_spot_check():
    """A seeded sample of the 37,500 config-2/3 list digests re-derived here
    (the full set is checked on the GPU in tests/test_gpu_configs.py)."""
    fx = load("cfg23_digests.json")
    rng = np.random.default_rng(23)
    for sigma in (2, 16, 128):
        t = inputs.config2_text(sigma)
        assert tdigest(t.tobytes()) == fx["texts"][f"cfg2_{sigma}"]
        for m in rng.choice(inputs.DEFAULT_LENGTHS, 3, replace=False):
            pats = inputs.config2_patterns(t, sigma, int(m))
            for k in rng.integers(0, 500, 2):
                r = oracle.search(pats[k], t, threads=4)
                assert [r.size, digest(r)] == fx["cfg2"][str(sigma)][str(m)][k], (sigma, m, k)
    assert sum(len(v) for c in fx["cfg2"].values() for v in c.values()) == 35000
    assert sum(len(v) for v in fx["cfg3"].values()) == 2500
