"""Seeded case generators mirrored from the reference test suite (test infra).

fuzz_cases      <- pkg/tests/conftest.py:35-58 (same draws, same order)
make_diff_case  <- pkg/src/matchbench/differential.py:70-92 (_make_case)
KNOWN           <- known-answer vectors of pkg/tests/test_*.py
"""
from __future__ import annotations

import math

import numpy as np

from paper_1012_2547_b200.inputs import ALLOWED_SIGMAS, derive_seed


def rand_bytes(rng, sigma: int, n: int) -> bytes:
    return rng.integers(0, sigma, size=n, dtype=np.uint8).tobytes()


def fuzz_cases(seed, count, m_lo, m_hi, *, sigmas=(1, 2, 4, 8, 32, 64, 128, 256), n_max=512, extract_prob=0.6):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        sigma = int(rng.choice(sigmas))
        m = int(rng.integers(m_lo, m_hi + 1))
        n = int(rng.integers(m, max(n_max, m) + 1))
        t = rand_bytes(rng, sigma, n)
        roll = rng.random()
        if roll < extract_prob:
            i = int(rng.integers(0, n - m + 1))
            p = t[i : i + m]
        elif roll < extract_prob + 0.2 or sigma == 1:
            p = rand_bytes(rng, sigma, m)
        else:
            i = int(rng.integers(0, n - m + 1))
            b = bytearray(t[i : i + m])
            j = int(rng.integers(0, m))
            b[j] = (b[j] + 1) % sigma
            p = bytes(b)
        yield p, t


KINDS = ("extracted", "random", "mutated")


def make_diff_case(m_min: int, m_max, case_seed: int, max_n: int = 4096):
    rng = np.random.Generator(np.random.PCG64(case_seed))
    sigma = int(rng.choice(ALLOWED_SIGMAS))
    lo = m_min
    hi = m_max if m_max is not None else max_n
    hi = min(hi, max_n)
    m = int(round(2 ** rng.uniform(math.log2(lo), math.log2(hi))))
    m = max(lo, min(m, hi))
    n = int(rng.integers(m, max_n + 1))
    text = rng.integers(0, sigma, size=n, dtype=np.uint8).tobytes()
    kind = KINDS[int(rng.integers(0, 3))]
    if kind == "random":
        pattern = rng.integers(0, sigma, size=m, dtype=np.uint8).tobytes()
    else:
        i = int(rng.integers(0, n - m + 1))
        pattern = text[i : i + m]
        if kind == "mutated":
            j = int(rng.integers(0, m))
            b = bytearray(pattern)
            b[j] = (b[j] + 1 + int(rng.integers(0, max(sigma - 1, 1)))) % sigma
            pattern = bytes(b)
    return sigma, n, m, kind, pattern, text


def diff_case_seed(seed, algo_id, i):
    return derive_seed(seed, algo_id, i)


# (pattern, text, expected) known answers from the reference tests
KNOWN = [
    (b"aba", b"ababa", [0, 2]),                      # test_core.py:38
    (b"b", b"aaaa", []),                             # test_core.py:39
    (b"abc", b"ab", []),                             # test_core.py:40 (m > n)
    (b"zz", b"abab", []),                            # test_comparison.py:24
    (b"ab", b"abab", [0, 2]),                        # test_comparison.py:33
    (b"abcab", b"abc", []),                          # test_comparison.py:34
    (b"abba", b"abba", [0]),                         # test_comparison.py:38
    (b"aa", b"bbbb", []),                            # test_comparison.py:39
    (b"aaa", b"aaaaa", [0, 1, 2]),                   # test_comparison.py:43
    (b"ab", b"ba", []),                              # test_comparison.py:44
    (b"abc", b"aabcc", [1]),                         # test_comparison.py:65
    (b"\x00" * 32, b"\x00" * 1024, list(range(993))),  # test_comparison.py:113-114
    (b"ab", b"abba", [0]),                           # test_bitparallel.py:119
    (b"x" * 63, b"x" * 100, list(range(38))),        # test_bitparallel.py:120
    (b"a" * 200, b"a" * 1000, list(range(801))),     # test_bitparallel.py:139-140
    (b"x" * 33, b"x" * 50, list(range(18))),         # test_registry.py:149
    (b"abc", b"abcabc", [0, 3]),                     # test_cli.py:141-149
    (b"a", b"", []),                                 # n = 0 is legal (test_core.py:20)
]
