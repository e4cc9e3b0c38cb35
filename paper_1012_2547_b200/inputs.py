"""Seeded synthetic inputs for the five BASELINE.json configs.

The generators of the reference benchmark harness are mirrored exactly
(pkg/src/matchbench/bench.py:80-155): blake2b-64 sub-seeds, numpy PCG64,
``integers(0, sigma, size, uint8)`` texts and uniform extraction offsets.
Configs 3 (Zipf natural-language-like) and 5 (dense 'a' adversarial) have no
reference generator; they follow SURVEY.md 8(d).  Large texts are generated in
chunks straight into a caller buffer (optionally pinned host memory) so that
16 GiB never needs a second copy.
"""
from __future__ import annotations

import hashlib

import numpy as np

PRNG_NAME = "numpy-pcg64"  # bench.py:27
ALLOWED_SIGMAS = (2, 4, 8, 16, 32, 64, 128, 256)  # bench.py:29
DEFAULT_LENGTHS = (2, 4, 8, 16, 32, 64, 128, 256, 512, 1024)  # bench.py:31
ROOT_SEED = 2026  # recorded root seed of every config


def derive_seed(*parts) -> int:
    """bench.py:80-83 -- stable 64-bit sub-seed."""
    h = hashlib.blake2b("|".join(str(p) for p in parts).encode(), digest_size=8)
    return int.from_bytes(h.digest(), "big")


def rand_text_np(sigma: int, size: int, seed: int, out: np.ndarray | None = None,
                 chunk: int = 1 << 28) -> np.ndarray:
    """bench.py:86-100 generate_rand_text bytes: PCG64(seed).integers(0, sigma, size, uint8).

    For sizes above `chunk` the stream is drawn in chunk-sized calls; numpy's
    uint8 draws consume whole 32-bit words per call, so chunk sizes that are
    multiples of 4 reproduce the single-call stream (tests/test_inputs.py)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if out is None:
        out = np.empty(size, dtype=np.uint8)
    pos = 0
    while pos < size:
        k = min(chunk, size - pos)
        out[pos : pos + k] = rng.integers(0, sigma, size=k, dtype=np.uint8)
        pos += k
    return out


def sample_positions(n: int, m: int, count: int, seed: int) -> list[int]:
    """bench.py:141-149 -- uniform extraction offsets in [0, n-m]."""
    if m > n:
        raise ValueError(f"cannot sample length-{m} patterns from a length-{n} text")
    if count < 1:
        raise ValueError("count must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, n - m + 1, size=count).tolist()


def sample_patterns(text: np.ndarray, m: int, count: int, seed: int) -> list[bytes]:
    """bench.py:152-155 -- patterns copied from the text at sample_positions."""
    return [text[i : i + m].tobytes() for i in sample_positions(text.size, m, count, seed)]


# ---- config generators ----

def config1(seed: int = ROOT_SEED):
    """1 MiB, sigma=4, one m=8 pattern extracted from the text."""
    n = 1 << 20
    t = rand_text_np(4, n, derive_seed(seed, "cfg1", "text"))
    pats = sample_patterns(t, 8, 1, derive_seed(seed, "cfg1", "pat"))
    return t, pats


def config2_text(sigma: int, seed: int = ROOT_SEED, n: int = 4 << 20):
    return rand_text_np(sigma, n, derive_seed(seed, "cfg2", "rand", sigma))


def config2_patterns(text: np.ndarray, sigma: int, m: int, count: int = 500, seed: int = ROOT_SEED):
    return sample_patterns(text, m, count, derive_seed(seed, "cfg2", sigma, m))


def zipf_text(n: int, seed: int, out: np.ndarray | None = None, chunk: int = 1 << 26) -> np.ndarray:
    """Config 3: bytes 0x20..0x7E, Zipf(s=1) by rank; space is rank 1, the other
    94 symbols ranked by a seeded permutation."""
    ranks = np.arange(1, 96, dtype=np.float64)
    prob = (1.0 / ranks) / np.sum(1.0 / ranks)
    rng = np.random.Generator(np.random.PCG64(seed))
    others = np.array([c for c in range(0x21, 0x7F)], dtype=np.uint8)
    perm = rng.permutation(others)
    symbols = np.concatenate([np.array([0x20], dtype=np.uint8), perm])
    if out is None:
        out = np.empty(n, dtype=np.uint8)
    pos = 0
    while pos < n:
        k = min(chunk, n - pos)
        out[pos : pos + k] = symbols[rng.choice(95, size=k, p=prob)]
        pos += k
    return out


def config3(seed: int = ROOT_SEED, n: int = 64 << 20):
    return zipf_text(n, derive_seed(seed, "cfg3", "text"))


def config3_patterns(text: np.ndarray, m: int, count: int = 500, seed: int = ROOT_SEED):
    return sample_patterns(text, m, count, derive_seed(seed, "cfg3", m))


STRIPE = 256 << 20  # config-4 text is generated in independent 256 MiB stripes


def config4_text(n: int = 16 << 30, seed: int = ROOT_SEED, out: np.ndarray | None = None,
                 threads: int | None = None) -> np.ndarray:
    """Config 4: i.i.d. uniform sigma=256.  Stripe i (256 MiB) is
    generate_rand_text(256, 256 MiB, derive_seed(seed, "cfg4", "text", i)) of the
    reference (bench.py:86-100); stripes are drawn in parallel threads (numpy
    releases the GIL), so 16 GiB takes seconds instead of a minute."""
    import concurrent.futures as cf
    import os

    if out is None:
        out = np.empty(n, dtype=np.uint8)
    nstripes = (n + STRIPE - 1) // STRIPE

    def one(i):
        lo = i * STRIPE
        hi = min(n, lo + STRIPE)
        rand_text_np(256, hi - lo, derive_seed(seed, "cfg4", "text", i), out=out[lo:hi])

    workers = threads or min(32, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(workers) as ex:
        list(ex.map(one, range(nstripes)))
    return out


def config4_patterns(text: np.ndarray, lengths=(2, 8, 32, 128, 1024), seed: int = ROOT_SEED):
    return [sample_patterns(text, m, 1, derive_seed(seed, "cfg4", m))[0] for m in lengths]


def dense_text(n: int, seed: int, out: np.ndarray | None = None) -> np.ndarray:
    """Config 5: 99.9% 'a'; 0.1% of positions (seeded, without replacement) set
    to bytes uniform over 'b'..'z'."""
    if out is None:
        out = np.empty(n, dtype=np.uint8)
    out[:] = ord("a")
    rng = np.random.Generator(np.random.PCG64(seed))
    k = n // 1000
    pos = rng.choice(n, size=k, replace=False) if n <= (1 << 24) else _sample_without_replacement(rng, n, k)
    out[pos] = rng.integers(ord("b"), ord("z") + 1, size=k, dtype=np.uint8)
    return out


def _sample_without_replacement(rng, n: int, k: int) -> np.ndarray:
    # k << n: draw with replacement, dedupe, top up (deterministic per seed)
    got = np.unique(rng.integers(0, n, size=k + k // 8 + 16))
    while got.size < k:
        got = np.unique(np.concatenate([got, rng.integers(0, n, size=k - got.size + 16)]))
    return np.sort(rng.permutation(got)[:k])


def config5(seed: int = ROOT_SEED, n: int = 256 << 20):
    return dense_text(n, derive_seed(seed, "cfg5", "text"))


def config5_patterns(lengths=(2, 16, 128, 1024)):
    pats = []
    for m in lengths:
        pats.append(b"a" * m)
        pats.append(b"a" * (m - 1) + b"b")
    return pats
