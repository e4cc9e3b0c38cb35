"""GPU-backed drop-ins for every searcher entry point of the reference.

Each ``compile_X(p)`` enforces X's applicability bounds exactly as the
reference does -- at compile time, before any scan (comparison.py:241-245,
317-318; bitparallel.py:91-92, 177-181, 225-226; automata.py:100-101) -- then
returns a ``run(hay) -> list[int]`` closure over one immutable engine plan.
All entry points compute the same function, so they share the
engine; the names differ only in their bounds.  ``run`` also accepts a uint8
CUDA tensor (zero copy) and rejects InstrumentedText (reads mode is a CPU
metric).
"""
from __future__ import annotations

from . import engine
from .core import WORD, ApplicabilityError, InstrumentedText, Text, WordSpec, as_haystack, as_needle

HASH_GRAM_LENGTHS = (3, 5, 8)  # comparison.py:224
SBNDM_GRAM_LENGTHS = (2, 4, 6, 8)  # bitparallel.py:171


def _len(hay) -> int:
    try:
        return int(hay.numel())  # torch tensor
    except AttributeError:
        return len(hay)


def compile_engine(p: bytes, family: str = "auto"):
    """The engine's own compile: plan once, return run(hay) -> list[int]."""
    plan = engine.Plan(p, family)
    m = plan.m

    def run(hay) -> list[int]:
        if isinstance(hay, InstrumentedText):
            raise TypeError("InstrumentedText (reads mode) is not supported by the GPU engine")
        hay = as_haystack(hay)
        if m > _len(hay):
            return []
        return engine.find(plan, hay).tolist()

    run.plan = plan
    return run


def compile_tensor(p: bytes, family: str = "auto"):
    """Like compile_engine but run(hay) returns the int64 CUDA tensor of positions."""
    plan = engine.Plan(p, family)

    def run(hay):
        return engine.find(plan, as_haystack(hay))

    run.plan = plan
    return run


def _bounded(name: str, lo: int = 1, hi: int | None = None, hi_label: str | None = None):
    def compile_fn(p: bytes, word: WordSpec = WORD):
        m = len(p)
        if m < lo:
            raise ApplicabilityError(name, m, f"m >= {lo}")
        if hi is not None:
            h = hi(word) if callable(hi) else hi
            if m > h:
                raise ApplicabilityError(name, m, hi_label.format(w=word.w, h=h))
        return compile_engine(p)

    compile_fn.__name__ = "compile_" + name.lower().replace("-", "_")
    return compile_fn


# comparison.py:70-221
compile_hor = _bounded("HOR")
compile_qs = _bounded("QS")
compile_br = _bounded("BR")
compile_tvsbs = _bounded("TVSBS")
compile_fjs = _bounded("FJS")


def compile_hashq(q: int, p: bytes):
    """comparison.py:234-245 bounds: q in (3, 5, 8) else ValueError; m >= q."""
    if q not in HASH_GRAM_LENGTHS:
        raise ValueError(f"q must be one of {HASH_GRAM_LENGTHS}, got {q}")
    if len(p) < q:
        raise ApplicabilityError(f"HASH{q}", len(p), f"m >= {q}")
    return compile_engine(p)


def compile_ssef(p: bytes, word: WordSpec = WORD):
    """comparison.py:308-318 bound: m >= 32."""
    if len(p) < 32:
        raise ApplicabilityError("SSEF", len(p), "m >= 32")
    return compile_engine(p)


# automata.py:59-141
compile_bom = _bounded("BOM")


def compile_ebom(p: bytes):
    """automata.py:92-101 bound: m >= 2."""
    if len(p) < 2:
        raise ApplicabilityError("EBOM", len(p), "m >= 2")
    return compile_engine(p)


# bitparallel.py:41-422
def compile_so(p: bytes, word: WordSpec = WORD):
    return compile_engine(p)


def compile_sa(p: bytes, word: WordSpec = WORD):
    return compile_engine(p)


compile_bndm = _bounded("BNDM", hi=lambda w: w.w, hi_label="m <= w ({w})")
compile_sbndm = _bounded("SBNDM", hi=lambda w: w.w, hi_label="m <= w ({w})")
compile_sbndm_bmh = _bounded("SBNDM-BMH", hi=lambda w: w.w, hi_label="m <= w ({w})")
compile_bmh_sbndm = _bounded("BMH-SBNDM", hi=lambda w: w.w, hi_label="m <= w ({w})")
compile_fsbndm = _bounded("FSBNDM", hi=lambda w: w.w - 1, hi_label="m <= w-1 ({h})")


def compile_sbndmq(q: int, p: bytes, word: WordSpec = WORD):
    """bitparallel.py:174-181 bounds: q in (2,4,6,8) else ValueError; q <= m <= w."""
    if q not in SBNDM_GRAM_LENGTHS:
        raise ValueError(f"q must be one of {SBNDM_GRAM_LENGTHS}, got {q}")
    m = len(p)
    if m < q:
        raise ApplicabilityError(f"SBNDMq{q}", m, f"m >= {q}")
    if m > word.w:
        raise ApplicabilityError(f"SBNDMq{q}", m, f"m <= w ({word.w})")
    return compile_engine(p)


def compile_lbndm(p: bytes, word: WordSpec = WORD):
    return compile_engine(p)


# ---- search_* wrappers (comparison.py:355-380, bitparallel.py:425-458, automata.py:144-149)
def search_hor(pattern, text) -> list[int]:
    return compile_hor(as_needle(pattern))(as_haystack(text))


def search_qs(pattern, text) -> list[int]:
    return compile_qs(as_needle(pattern))(as_haystack(text))


def search_br(pattern, text) -> list[int]:
    return compile_br(as_needle(pattern))(as_haystack(text))


def search_tvsbs(pattern, text) -> list[int]:
    return compile_tvsbs(as_needle(pattern))(as_haystack(text))


def search_fjs(pattern, text) -> list[int]:
    return compile_fjs(as_needle(pattern))(as_haystack(text))


def search_hashq(q: int, pattern, text) -> list[int]:
    return compile_hashq(q, as_needle(pattern))(as_haystack(text))


def search_ssef(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_ssef(as_needle(pattern), word)(as_haystack(text))


def search_bom(pattern, text) -> list[int]:
    return compile_bom(as_needle(pattern))(as_haystack(text))


def search_ebom(pattern, text) -> list[int]:
    return compile_ebom(as_needle(pattern))(as_haystack(text))


def search_so(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_so(as_needle(pattern), word)(as_haystack(text))


def search_sa(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_sa(as_needle(pattern), word)(as_haystack(text))


def search_bndm(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_bndm(as_needle(pattern), word)(as_haystack(text))


def search_sbndm(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_sbndm(as_needle(pattern), word)(as_haystack(text))


def search_sbndmq(q: int, pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_sbndmq(q, as_needle(pattern), word)(as_haystack(text))


def search_fsbndm(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_fsbndm(as_needle(pattern), word)(as_haystack(text))


def search_lbndm(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_lbndm(as_needle(pattern), word)(as_haystack(text))


def search_sbndm_bmh(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_sbndm_bmh(as_needle(pattern), word)(as_haystack(text))


def search_bmh_sbndm(pattern, text, word: WordSpec = WORD) -> list[int]:
    return compile_bmh_sbndm(as_needle(pattern), word)(as_haystack(text))


def search(pattern, text) -> list[int]:
    """Engine-native convenience: all positions as list[int]."""
    return compile_engine(as_needle(pattern))(as_haystack(text))


def count(pattern, text) -> int:
    """Engine-native occurrence count (no positions written)."""
    p = as_needle(pattern)
    hay = as_haystack(text)
    if isinstance(hay, InstrumentedText):
        raise TypeError("InstrumentedText (reads mode) is not supported by the GPU engine")
    if len(p) > _len(hay):
        return 0
    return engine.count(engine.Plan(p), hay)


def search_many(patterns, text):
    """Batched mode (one launch): list of list[int], one per pattern, in order."""
    pats = [as_needle(p) for p in patterns]
    hay = as_haystack(text)
    if not pats:
        return []
    plans = [engine.Plan(p) for p in pats]
    pos, offs = engine.find_batch(plans, hay)
    host = pos.cpu()
    o = offs.tolist()
    return [host[o[k] : o[k + 1]].tolist() for k in range(len(pats))]
