"""Generate the golden fixtures of tests/golden/ by running the REFERENCE itself.

Run in the build container, where the read-only reference is importable:

    python tests/golden/make_golden.py            # writes tests/golden/*.json

Nothing else reads /root/reference: the GPU box never has it, so the tests use
only the committed JSON.  Every expected result below comes from the
reference's own functions (matchbench.core.brute_force_search, search_so,
the table builders, conftest.fuzz_cases, differential._make_case,
bench.generate_rand_text / sample_positions), so these fixtures pin both the
oracle restatement (oracle/oracle.c) and the case/input generator mirrors
(tests/cases.py, paper_1012_2547_b200/inputs.py).
"""
from __future__ import annotations

import hashlib
import importlib.util
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from matchbench import bench as rbench  # noqa: E402
from matchbench import bitparallel as rbp  # noqa: E402
from matchbench import comparison as rcmp  # noqa: E402
from matchbench import differential as rdiff  # noqa: E402
from matchbench.core import brute_force_search  # noqa: E402
from matchbench.registry import REGISTRY  # noqa: E402

spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(REF, "tests", "conftest.py"))
ref_conftest = importlib.util.module_from_spec(spec)
spec.loader.exec_module(ref_conftest)

from paper_1012_2547_b200 import inputs  # noqa: E402  (config 3/5 generators have no reference twin)


def digest(pos) -> str:
    return hashlib.sha1(np.asarray(pos, dtype="<i8").tobytes()).hexdigest()[:16]


def tdigest(b: bytes) -> str:
    return hashlib.sha1(b).hexdigest()[:16]


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
    print("wrote", name)


def tables():
    rng = np.random.default_rng(4242)
    rows = []
    for _ in range(60):
        m = int(rng.integers(1, 130))
        sigma = int(rng.choice([1, 2, 4, 256]))
        p = rng.integers(0, sigma, size=m, dtype=np.uint8).tobytes()
        fm = rbp.forward_masks(p)
        rows.append({
            "p": p.hex(),
            "hor": rcmp._horspool_table(p),
            "sun": rcmp._sunday_table(p),
            "kmp": rcmp.kmp_failure(p),
            "fwd": {str(c): hex(v) for c, v in enumerate(fm) if v},
            "gram": {str(q): [rcmp._gram_hash(p, i, q) for i in range(m - q + 1)] for q in (3, 5, 8) if m >= q},
        })
    dump("tables.json", rows)


def fuzz():
    sets = [
        dict(seed=11, count=300, m_lo=1, m_hi=64, n_max=2048),
        dict(seed=101, count=200, m_lo=3, m_hi=256, n_max=1024),
        dict(seed=13, count=150, m_lo=32, m_hi=1024, n_max=4096, sigmas=(2, 4, 64)),
        dict(seed=40, count=120, m_lo=65, m_hi=1024, n_max=4096),
        dict(seed=21, count=200, m_lo=1, m_hi=8, n_max=512),
    ]
    out = []
    for s in sets:
        kw = {k: v for k, v in s.items() if k not in ("seed", "count", "m_lo", "m_hi")}
        cases = []
        for p, t in ref_conftest.fuzz_cases(s["seed"], s["count"], s["m_lo"], s["m_hi"], **kw):
            r = brute_force_search(p, t)
            cases.append([len(p), len(t), tdigest(p + b"|" + t), len(r), digest(r)])
        out.append({"params": s, "cases": cases})
    dump("fuzz.json", out)


def differential():
    seed, total = 2026, 10000
    per_algo = -(-total // len(REGISTRY))
    rows = {}
    for algo in REGISTRY:
        lst = []
        for i in range(per_algo):
            cs = rbench.derive_seed(seed, algo.id, i)
            sigma, n, m, kind, pattern, text = rdiff._make_case(algo, cs, rdiff.DEFAULT_MAX_N)
            r = brute_force_search(pattern, text)
            lst.append([sigma, n, m, kind[0], len(r), digest(r)])
        rows[algo.id] = {"m_min": algo.m_min, "m_max": algo.m_max, "cases": lst}
    dump("differential.json", {"seed": seed, "per_algo": per_algo, "algos": rows})


def configs():
    res = {}
    # config 1 -- reference generators end to end
    n1 = 1 << 20
    s_text = inputs.derive_seed(inputs.ROOT_SEED, "cfg1", "text")
    s_pat = inputs.derive_seed(inputs.ROOT_SEED, "cfg1", "pat")
    t1 = rbench.generate_rand_text(4, n1, s_text)
    (p1,) = rbench.sample_patterns(t1, 8, 1, s_pat)
    r1 = brute_force_search(p1, t1)
    res["cfg1"] = {"text": tdigest(t1.data), "pattern": p1.data.hex(), "positions": r1}
    # config 2 -- 4 MiB texts per sigma, first 2 of 500 patterns per cell
    cells = []
    for sigma in (2, 4, 8, 16, 32, 64, 128):
        t = rbench.generate_rand_text(sigma, 4 << 20, inputs.derive_seed(inputs.ROOT_SEED, "cfg2", "rand", sigma))
        for m in (2, 4, 8, 16, 32, 64, 128, 256, 512, 1024):
            offs = rbench.sample_positions(t, m, 500, inputs.derive_seed(inputs.ROOT_SEED, "cfg2", sigma, m))
            for i in offs[:2]:
                p = t.data[i : i + m]
                r = brute_force_search(p, t)
                cells.append([sigma, m, i, len(r), digest(r)])
        cells.append([sigma, 0, 0, 0, tdigest(t.data)])
        print("cfg2 sigma", sigma, flush=True)
    res["cfg2"] = cells
    # config 3 -- Zipf text, 4 MiB prefix of the 64 MiB stream (chunked generator)
    t3 = inputs.zipf_text(4 << 20, inputs.derive_seed(inputs.ROOT_SEED, "cfg3", "text"))
    rows3 = []
    for m in (4, 16, 64, 256, 1024):
        offs = rbench.sample_positions(rbench.Text(t3.tobytes()), m, 3, inputs.derive_seed(inputs.ROOT_SEED, "cfg3p", m))
        for i in offs:
            p = t3[i : i + m].tobytes()
            r = brute_force_search(p, t3.tobytes())
            rows3.append([m, i, len(r), digest(r)])
    res["cfg3_4MiB"] = {"text": tdigest(t3.tobytes()), "rows": rows3}
    # config 4 -- 4 MiB prefix of the sigma=256 stream
    t4 = rbench.generate_rand_text(256, 4 << 20, inputs.derive_seed(inputs.ROOT_SEED, "cfg4", "text", 0))
    rows4 = []
    for m in (2, 8, 32, 128, 1024):
        (i,) = rbench.sample_positions(t4, m, 1, inputs.derive_seed(inputs.ROOT_SEED, "cfg4p", m))
        p = t4.data[i : i + m]
        r = brute_force_search(p, t4)
        rows4.append([m, i, len(r), digest(r)])
    res["cfg4_4MiB"] = {"text": tdigest(t4.data), "rows": rows4}
    # config 5 -- 4 MiB dense text; oracle = search_so (BF is O(n*m) here)
    t5 = inputs.dense_text(4 << 20, inputs.derive_seed(inputs.ROOT_SEED, "cfg5", "text"))
    rows5 = []
    for p in inputs.config5_patterns():
        r = rbp.search_so(p, t5.tobytes())
        rows5.append([p.hex(), len(r), digest(r)])
        print("cfg5", len(p), len(r), flush=True)
    res["cfg5_4MiB"] = {"text": tdigest(t5.tobytes()), "rows": rows5}
    dump("configs.json", res)


if __name__ == "__main__":
    what = sys.argv[1:] or ["tables", "fuzz", "differential", "configs"]
    for w in what:
        globals()[w]()
