"""Reference-signature harness helpers around the GPU engine.

Same names and argument meanings as the reference's benchmark module
(pkg/src/matchbench/bench.py:41-238) and bit-parallel helpers, so code that
generates inputs or times searchers through matchbench keeps working:
``generate_rand_text`` / ``sample_positions`` / ``sample_patterns`` /
``standard_texts`` return the reference's types and byte streams;
``run_benchmark`` runs the reference's time-mode protocol with every search
timed by CUDA events on the GPU ("reads" mode counts CPU character reads and
is rejected).
"""
from __future__ import annotations

import statistics
import warnings
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .core import WORD, Pattern, Text, WordSpec
from .inputs import ALLOWED_SIGMAS, DEFAULT_LENGTHS, PRNG_NAME, derive_seed, rand_text_np

FULL_TEXT_SIZE = 5 * 2**20  # bench.py:34
DESK_TEXT_SIZE = 2**20      # bench.py:36
METRICS = ("time", "reads")


def state_word_count(m: int, word: WordSpec = WORD) -> int:
    """bitparallel.py:19-21."""
    return -(-m // word.w)


def generate_rand_text(sigma: int, size: int, seed: int, allow_any_sigma: bool = False) -> Text:
    """bench.py:86-100: uniform i.i.d. bytes over 0..sigma-1 (numpy PCG64)."""
    if not allow_any_sigma and sigma not in ALLOWED_SIGMAS:
        raise ValueError(f"sigma must be one of {ALLOWED_SIGMAS} (or pass allow_any_sigma=True)")
    if not 1 <= sigma <= 256:
        raise ValueError(f"sigma must be in [1, 256], got {sigma}")
    if size < 1:
        raise ValueError("size must be >= 1")
    return Text(rand_text_np(sigma, size, seed).tobytes(), f"rand{sigma}")


def sample_positions(text: Text, m: int, count: int, seed: int) -> list[int]:
    """bench.py:141-149."""
    n = len(text)
    if m > n:
        raise ValueError(f"cannot sample length-{m} patterns from a length-{n} text")
    if count < 1:
        raise ValueError("count must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, n - m + 1, size=count).tolist()


def sample_patterns(text: Text, m: int, count: int, seed: int) -> list[Pattern]:
    """bench.py:152-155."""
    return [Pattern(text.data[i : i + m]) for i in sample_positions(text, m, count, seed)]


@dataclass(frozen=True)
class BenchConfig:
    """bench.py:41-61 (same fields and validation)."""

    lengths: tuple = DEFAULT_LENGTHS
    patterns_per_length: int = 400
    seed: int = 1
    metric: str = "time"
    text_size: int = FULL_TEXT_SIZE
    warmup: bool = True

    def __post_init__(self):
        object.__setattr__(self, "lengths", tuple(self.lengths))
        if any(b <= a for a, b in zip(self.lengths, self.lengths[1:])):
            raise ValueError("lengths must be strictly increasing")
        if not self.lengths:
            raise ValueError("lengths must be non-empty")
        if self.patterns_per_length < 1:
            raise ValueError("patterns_per_length must be >= 1")
        if self.metric not in METRICS:
            raise ValueError(f"metric must be one of {METRICS}")
        if self.text_size < 1:
            raise ValueError("text_size must be >= 1")


@dataclass(frozen=True)
class Measurement:
    """bench.py:64-77: one benchmark cell (mean over patterns)."""

    text_id: str
    sigma: int
    family: str
    algorithm: str
    m: int
    runs: int
    mean_value: float  # milliseconds (CUDA events)
    stddev: float
    mean_occurrences: float
    metric: str


def standard_texts(cfg: BenchConfig, sigmas=ALLOWED_SIGMAS) -> list[Text]:
    """bench.py:158-164."""
    return [generate_rand_text(s, cfg.text_size, derive_seed(cfg.seed, "rand", s)) for s in sigmas]


#: bench.py:104-109 -- (bytes, approximate distinct symbols) of the paper's corpora
CORPUS_EXPECTATIONS = {
    "ecoli": (4_638_690, 4),
    "bible": (4_047_392, 63),
    "world192": (2_473_400, 94),
    "hs": (3_295_751, 20),
}


def load_corpus(path, expected_id: str | None = None) -> Text:
    """bench.py:112-138: a corpus file as raw bytes.  For the known corpus ids
    a length or alphabet that differs from the expectation only warns (corpus
    editions vary); sigma is counted on the device (K0 histogram)."""
    path = Path(path)
    data = path.read_bytes()
    text = Text(data, expected_id or path.stem)
    exp = CORPUS_EXPECTATIONS.get(text.id)
    if exp is not None:
        exp_n, exp_sigma = exp
        if len(data) != exp_n:
            warnings.warn(f"corpus {text.id!r}: expected n={exp_n:,} bytes, got {len(data):,} (different edition?)",
                          stacklevel=2)
        sigma = text.alphabet_size()
        if abs(sigma - exp_sigma) > 2:
            warnings.warn(f"corpus {text.id!r}: expected sigma~{exp_sigma}, got {sigma}", stacklevel=2)
    return text


def run_benchmark(cfg: BenchConfig, texts, algos=None, parallel: bool = False) -> list[Measurement]:
    """bench.py:204-238 cells, each search timed on the GPU (compile untimed, one
    warm-up, CUDA events around the search, mean/pstdev over the patterns)."""
    from .cli import gpu_benchmark
    from .registry import REGISTRY

    if cfg.metric != "time":
        raise ValueError("reads mode counts CPU character reads; the GPU engine supports metric='time'")
    if parallel:
        raise ValueError("parallel runs are only allowed in reads mode")
    algos = list(REGISTRY) if algos is None else list(algos)
    if not texts or not algos:
        raise ValueError("need at least one text and one algorithm")
    out = []
    for text in texts:
        rows = gpu_benchmark(text.data, text.id, algos, cfg.lengths, cfg.patterns_per_length, cfg.seed,
                             warmup=cfg.warmup)
        for r in rows:
            out.append(Measurement(r[0], r[1], r[2], r[3], r[4], cfg.patterns_per_length, r[5], r[6], r[7], r[8]))
    return out


__all__ = ["ALLOWED_SIGMAS", "CORPUS_EXPECTATIONS", "DEFAULT_LENGTHS", "PRNG_NAME", "BenchConfig", "Measurement",
           "derive_seed", "load_corpus",
           "generate_rand_text", "run_benchmark", "sample_patterns", "sample_positions", "standard_texts",
           "state_word_count"]
