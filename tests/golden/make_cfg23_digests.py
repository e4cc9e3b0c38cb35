"""Occurrence-list digests of EVERY config-2 and config-3 pattern (37,500 lists).

    python tests/golden/make_cfg23_digests.py     # writes tests/golden/cfg23_digests.json

Expected results come from the C oracle's brute force (oracle/oracle.c
orc_bf, a restatement of core.py:139-161 pinned against the reference itself by
tests/golden/{differential,fuzz,configs}.json).  Per pattern: the occurrence
count and sha1(int64 little-endian positions)[:16], the same digest the other
golden files use.  Identical patterns of a cell are searched once.  Texts are
pinned by their own digests so a GPU box that generates different bytes fails
loudly instead of comparing against the wrong lists.

Runs on the CPU in a few minutes (threads over patterns; the oracle releases
the GIL).  Nothing on the product path reads this file.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1012_2547_b200 import inputs  # noqa: E402

CFG3_LENGTHS = (4, 16, 64, 256, 1024)


def digest(pos: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(pos, dtype="<i8").tobytes()).hexdigest()[:16]


def cell_rows(t: np.ndarray, pats: list[bytes], pool) -> list[list]:
    uniq = {}
    for p in pats:
        uniq.setdefault(p, None)

    def one(p):
        r = oracle.search(p, t, "BF", threads=1)
        return p, [int(r.size), digest(r)]

    for p, row in pool.map(one, list(uniq)):
        uniq[p] = row
    return [uniq[p] for p in pats]


def main():
    workers = os.cpu_count() or 4
    out = {"digest": "sha1(int64 LE positions)[:16]", "oracle": "oracle/oracle.c orc_bf (core.py:139-161)",
           "cfg2": {}, "cfg3": {}, "texts": {}}
    t0 = time.time()
    with cf.ThreadPoolExecutor(workers) as pool:
        for sigma in (2, 4, 8, 16, 32, 64, 128):
            t = inputs.config2_text(sigma)
            out["texts"][f"cfg2_{sigma}"] = hashlib.sha1(t.tobytes()).hexdigest()[:16]
            cells = {}
            for m in inputs.DEFAULT_LENGTHS:
                cells[str(m)] = cell_rows(t, inputs.config2_patterns(t, sigma, m), pool)
            out["cfg2"][str(sigma)] = cells
            print(f"cfg2 sigma={sigma} done {time.time() - t0:.0f}s", flush=True)
        t = inputs.config3()
        out["texts"]["cfg3"] = hashlib.sha1(t.tobytes()).hexdigest()[:16]
        for m in CFG3_LENGTHS:
            out["cfg3"][str(m)] = cell_rows(t, inputs.config3_patterns(t, m), pool)
            print(f"cfg3 m={m} done {time.time() - t0:.0f}s", flush=True)
    with open(os.path.join(HERE, "cfg23_digests.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"), sort_keys=True)
    n = sum(len(v) for c in out["cfg2"].values() for v in c.values()) + sum(len(v) for v in out["cfg3"].values())
    print(f"wrote cfg23_digests.json: {n} lists in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
