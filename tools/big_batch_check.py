"""Robustness: a 20,000-pattern batch on a 1 MiB sigma=16 text, sampled against the oracle (tools only)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle
import paper_1012_2547_b200 as mb
rng = np.random.default_rng(1)
t = rng.integers(0, 16, 1 << 20, dtype=np.uint8).tobytes()
pats = [t[i:i + m] for i, m in zip(rng.integers(0, len(t) - 64, 20000), rng.integers(2, 64, 20000))]
t0 = time.time(); res = mb.search_many(pats, t); dt = time.time() - t0
bad = sum(1 for k in range(0, 20000, 97) if res[k] != oracle.search(pats[k], t).tolist())
print("K=20000 done in %.2fs, checked %d, bad %d, total %d" % (dt, len(range(0, 20000, 97)), bad, sum(map(len, res))))
