"""CPU: the C-ABI library loads and exports every declared symbol; the host-side
mirror of the reference interface (bounds, errors, registry, selection map,
inputs, sharding) behaves like the reference -- no GPU compute here."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1012_2547_b200 as mb
from paper_1012_2547_b200 import engine, inputs, registry, searchers
from paper_1012_2547_b200.core import ApplicabilityError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "matchb200.h")).read()
    declared = set(re.findall(r"\b(mb_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(engine.EXPORTS)
    lib = ctypes.CDLL(engine.LIB_PATH)
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert b"sm_100a" in engine.load_library().mb_version()


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", engine.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_on_product_path():
    pkg = os.path.join(ROOT, "paper_1012_2547_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), fn
                assert "liboracle" not in src, fn


def test_search_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        mb.search_hor(b"ab", b"abab")


def test_bounds_and_errors_mirror_reference():
    # ApplicabilityError at compile time, with the reference's message format (core.py:23)
    with pytest.raises(ApplicabilityError, match=r"SSEF is not applicable at m=16: requires m >= 32"):
        mb.search_ssef(b"x" * 16, b"whatever")
    with pytest.raises(ApplicabilityError, match="m >= 32"):
        searchers.compile_ssef(b"x" * 31)
    with pytest.raises(ApplicabilityError):
        mb.search_hashq(5, b"abcd", b"whatever")
    with pytest.raises(ValueError):
        mb.search_hashq(4, b"abcd", b"whatever")
    with pytest.raises(ApplicabilityError, match=r"requires m <= w \(64\)"):
        mb.search_bndm(b"x" * 65, b"whatever")
    with pytest.raises(ApplicabilityError, match=r"m <= w-1 \(63\)"):
        mb.search_fsbndm(b"x" * 64, b"whatever")
    with pytest.raises(ApplicabilityError):
        mb.search_sbndmq(8, b"abcd", b"whatever")
    with pytest.raises(ValueError):
        mb.search_sbndmq(3, b"abc", b"whatever")
    with pytest.raises(ApplicabilityError):
        mb.search_ebom(b"a", b"aaa")
    with pytest.raises(ValueError):
        mb.brute_force_search(b"", b"abc")
    with pytest.raises(ValueError):
        mb.Pattern(b"")
    e = ApplicabilityError("X", 3, "m >= 5")
    assert isinstance(e, ValueError) and (e.algorithm, e.m, e.bound) == ("X", 3, "m >= 5")
    w32 = registry.build_registry(mb.WordSpec(32))
    d = {a.id: a for a in w32}
    assert d["BNDM"].m_max == 32 and d["FSBNDM"].m_max == 31
    with pytest.raises(ApplicabilityError):
        d["BNDM"].compile(b"x" * 33)


def test_registry_mirror():
    ids = [a.id for a in mb.REGISTRY]
    assert ids == ["HOR", "QS", "BR", "TVSBS", "FJS", "HASH3", "HASH5", "HASH8", "SSEF", "BOM", "EBOM", "SO",
                   "SA", "BNDM", "SBNDM", "LBNDM", "SBNDM-BMH", "BMH-SBNDM", "FSBNDM", "SBNDMq2", "SBNDMq4",
                   "SBNDMq6", "SBNDMq8"]
    assert "B200" not in ids and mb.get_algorithm("b200") is mb.B200
    assert mb.get_algorithm("hor").id == "HOR"
    with pytest.raises(KeyError):
        mb.get_algorithm("nope")
    assert {a.id for a in mb.applicable_algorithms(4)} >= {"HOR", "SO", "SA", "BNDM", "HASH3", "SBNDMq4"}
    assert not any(a.needs_word for a in mb.applicable_algorithms(2048))
    with pytest.raises(ValueError):
        mb.applicable_algorithms(0)


def test_selection_map_matches_reference_cells():
    sel = mb.select_applicable
    # SURVEY.md 8(d) auto-path picks
    assert [sel(256, m).id for m in (2, 8, 32, 128, 1024)] == ["FJS", "EBOM", "EBOM", "SSEF", "LBNDM"]
    assert [sel(95, m).id for m in (4, 16, 64, 256, 1024)] == ["FJS", "EBOM", "TVSBS", "TVSBS", "SSEF"]
    assert sel(4, 8).id == "HASH5"
    assert mb.classify(128, 4) == mb.SizeClasses("very_large", "very_short")
    csv = mb.DEFAULT_SELECTION_MAP.to_csv().strip().splitlines()
    assert len(csv) == 17 and "very_small,short,HASH5,derived-fill" in csv


def test_descriptor_substitution_seam():
    from dataclasses import replace

    gpu = replace(mb.get_algorithm("HOR"), id="B200-HOR", compile=searchers.compile_engine)
    assert gpu.id == "B200-HOR" and gpu.m_min == 1 and gpu.applicable(5000)
    wrapped = registry.b200_descriptor_for(mb.get_algorithm("SSEF"))
    with pytest.raises(ApplicabilityError):
        wrapped.compile(b"x" * 5)


def test_plan_info_families():
    cases = {1: "swar", 3: "swar", 4: "win4", 6: "win4", 7: "aligned", 64: "aligned", 65: "aligned",
             271: "aligned", 1024: "sampled", 8192: "sampled"}
    rng0 = np.random.default_rng(0)
    for m, fam in cases.items():
        assert engine.Plan(rng0.integers(0, 256, m, dtype=np.uint8).tobytes()).info().family == fam, m
    # rare byte confined to one gram (a^(m-1)b, b a^(m-1)): one-gram WIN4 anchor beats ALIGNED
    for m in (16, 128, 1024, 8192):
        assert engine.Plan(b"\x05" * (m - 1) + b"\x07").info().family == "win4", m
        assert engine.Plan(b"\x07" + b"\x05" * (m - 1)).info().family == "win4", m
    assert engine.Plan(b"a" * 100).info().periodic
    # small alphabets: exact SWAR at m = 5..7 instead of a busy anchor filter, K2 from m = 8
    for m, fam in ((5, "swar"), (6, "swar"), (7, "swar"), (8, "shiftor")):
        assert engine.Plan(bytes(rng0.integers(0, 2, m, dtype=np.uint8))).info().family == fam, m
    assert engine.Plan(bytes(range(40, 48))).info().family == "aligned"
    # sampled (K3) only for periods >= 294: a 256 KiB unit's occurrences fit its list
    unit = bytes(rng0.integers(0, 256, 200, dtype=np.uint8))
    assert engine.Plan((unit * 6)[:1024]).info().family != "sampled"
    unit = bytes(rng0.integers(0, 256, 300, dtype=np.uint8))
    assert engine.Plan((unit * 4)[:1024]).info().family == "sampled"
    assert not engine.Plan(b"a" * 99 + b"b").info().periodic
    with pytest.raises(ValueError):
        engine.Plan(b"x" * 8193)
    with pytest.raises(ValueError):
        engine.Plan(b"abc", family="aligned")
    # anchor choice keeps the rare byte of a^(m-1)b inside the anchor window
    info = engine.Plan(b"a" * 127 + b"b").info()
    assert info.anchor <= 127 <= info.anchor + 3
    rng = np.random.default_rng(1)
    long_random = rng.integers(0, 256, 1024, dtype=np.uint8).tobytes()
    assert engine.Plan(long_random).info().family == "sampled"
    assert engine.Plan(long_random[:271]).info().family == "aligned"
    assert engine.Plan(b"ab" * 512).info().family == "aligned"  # periodic: full scan
    assert engine.Plan(long_random, family="aligned").info().family == "aligned"
    with pytest.raises(ValueError):
        engine.Plan(b"a" * 1024, family="sampled")
    # K2 (bit-plane Shift-And): auto for binary texts at 8 <= m <= 22 and 3-4-letter ones at 8 <= m <= 14,
    # where the word filters are busy; longer patterns take the strided gram filter
    assert engine.Plan(bytes(rng.integers(0, 4, 40, dtype=np.uint8))).info().family == "gram"
    assert engine.Plan(bytes([0, 1, 1, 0, 1, 0, 0, 0, 1, 1, 1, 0])).info().family == "shiftor"
    assert engine.Plan(bytes([0, 1, 2, 3, 1, 0, 2, 2, 3, 1, 0, 3])).info().family == "shiftor"
    assert engine.Plan(bytes([0, 1, 1, 0, 1, 0])).info().family == "swar"  # m = 6: exact SWAR stays
    # K1G strided gram filter: small alphabets from m = 15 (S = 8) / 23 (S = 16); sigma >= 16 keeps ALIGNED
    i4 = engine.Plan(bytes(rng.integers(0, 4, 64, dtype=np.uint8))).info()
    assert (i4.family, i4.stride, i4.gram, i4.delta) == ("gram", 16, 16, 15)
    i8 = engine.Plan(bytes(rng.integers(0, 8, 16, dtype=np.uint8))).info()
    assert (i8.family, i8.stride, i8.gram, i8.delta) == ("gram", 8, 8, 7)
    assert engine.Plan(bytes(rng.integers(0, 16, 64, dtype=np.uint8))).info().family == "aligned"
    assert engine.Plan(bytes(rng.integers(0, 4, 12, dtype=np.uint8)), family="aligned").info().words == 2
    assert engine.Plan(b"ab" * 20).info().family == "aligned"  # periodic: break-run verification
    assert engine.Plan(bytes(rng.integers(0, 256, 15, dtype=np.uint8)), family="gram").info().family == "gram"
    with pytest.raises(ValueError):
        engine.Plan(bytes(14), family="gram")
    assert engine.Plan(bytes(rng.integers(0, 4, 40, dtype=np.uint8)), family="shiftor").info().family == "shiftor"
    with pytest.raises(ValueError):
        engine.Plan(b"x" * 65, family="shiftor")


def test_text_histogram_steers_small_alphabet_plans():
    """With the text's byte histogram (mb_plan_opts.hist, K0 on the device) the
    planner knows a 4-letter text from a 16-letter one: exact SWAR at m = 5..7
    and K2 from m = 8 over <= 4 letters, WIN4 / one-word ALIGNED over 16."""
    rng = np.random.default_rng(11)
    h4 = np.zeros(256, dtype=np.int64)
    h4[:4] = 1 << 20
    h16 = np.zeros(256, dtype=np.int64)
    h16[:16] = 1 << 18
    for m, fam4, fam16 in ((5, "swar", "win4"), (6, "swar", "win4"), (7, "swar", "aligned"), (8, "shiftor", "aligned"),
                           (12, "shiftor", "aligned")):
        p = bytes(rng.permutation(4)[np.arange(m) % 4].astype(np.uint8))  # 4 distinct letters, no short period
        p = p[:-1] + bytes([p[-1] ^ 1])
        assert engine.Plan(p, hist=h4).info().family == fam4, (m, "sigma 4")
        assert engine.Plan(p, hist=h16).info().family == fam16, (m, "sigma 16")
    assert engine.Plan(bytes([0, 1, 2, 3, 1, 0, 2, 2, 3, 1, 0, 3]), hist=h4).info().words == 2  # K2: two planes over 4 letters


def test_aligned_anchor_words():
    """The ALIGNED family widens its anchor to 2 words (11-byte window) over
    small alphabets (auto plans take K2 or the strided gram filter there);
    large alphabets keep one word; forced values are validated."""
    rng = np.random.default_rng(3)
    for sigma, words in ((2, 2), (4, 2), (64, 1), (256, 1)):
        p = rng.integers(0, sigma, 14 if sigma <= 4 else 64, dtype=np.uint8).tobytes()
        info = engine.Plan(p, family="aligned" if sigma <= 4 else "auto").info()
        assert (info.family, info.words) == ("aligned", words), sigma
    p = rng.integers(0, 256, 40, dtype=np.uint8).tobytes()
    for nw in (1, 2, 3):
        assert engine.Plan(p, anchor_words=nw).info().words == nw
    with pytest.raises(ValueError):
        engine.Plan(p[:10], anchor_words=2)   # window 11 > m
    with pytest.raises(ValueError):
        engine.Plan(p, anchor_words=4)
    assert engine.Plan(p[:4]).info().words == 0  # not ALIGNED


def test_inputs_mirror_reference_generators():
    rng_bytes = np.random.Generator(np.random.PCG64(7)).integers(0, 4, size=10007, dtype=np.uint8)
    assert np.array_equal(inputs.rand_text_np(4, 10007, 7, chunk=4096), rng_bytes)
    assert inputs.sample_positions(1000, 10, 3, 5) == np.random.Generator(np.random.PCG64(5)).integers(0, 991, size=3).tolist()
    assert inputs.derive_seed(1, "rand", 4) == inputs.derive_seed("1", "rand", "4")
    t = inputs.dense_text(100000, 3)
    assert (t != ord("a")).sum() == 100 and t.max() <= ord("z")
    z = inputs.zipf_text(200000, 3)
    assert z.min() >= 0x20 and z.max() <= 0x7E and abs((z == 0x20).mean() - 0.195) < 0.01


def _shard_worker(rank, world, port, text, pats, q):
    import torch.distributed as dist

    import oracle
    from paper_1012_2547_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for p in pats:
        lo, hi, rhi = shard.shard_bounds(len(text), len(p), world, rank)
        local, off, total = shard.sharded_search(p, text[lo:rhi], len(text), lambda a, b: oracle.search(a, b))
        res.append((rank, off, total, local.tolist()))
    q.put(res)
    dist.destroy_process_group()


def _shard_batch_worker(rank, world, port, text, pats, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1012_2547_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def batch(ps, t):  # the oracle stands in for engine.find_batch on this CPU test
        res = [oracle.search(p, t) for p in ps]
        offs = np.concatenate([[0], np.cumsum([r.size for r in res])])
        return np.concatenate(res) if res else np.zeros(0, np.int64), offs

    pos, offs = shard.sharded_search_batch(pats, text, batch)
    # text striping: every rank's slice of one pattern gathered into the global list
    p = pats[0]
    lo, hi, rhi = shard.shard_bounds(len(text), len(p), world, rank)
    local, _, _ = shard.sharded_search(p, text[lo:rhi], len(text), lambda a, b: oracle.search(a, b))
    full = shard.gather_positions(torch.from_numpy(np.asarray(local, dtype=np.int64)))
    q.put((rank, pos.tolist(), offs.tolist(), full.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batch_and_gather_gloo(world):
    """pattern-sharded batches (text replicated) gather into the
    batch CSR, and text-striped positions gather into the global list."""
    import multiprocessing as mp
    import socket

    import oracle

    rng = np.random.default_rng(10 + world)
    text = rng.integers(0, 4, 6000, dtype=np.uint8).tobytes()
    pats = [text[i : i + m] for i, m in zip(rng.integers(0, 5900, 7), (2, 3, 5, 8, 13, 40, 90))]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_batch_worker, args=(r, world, port, text, pats, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    want = [oracle.search(p, text).tolist() for p in pats]
    for rank, pos, offs, full in outs:
        for k in range(len(pats)):
            assert pos[offs[k] : offs[k + 1]] == want[k], (rank, k)
        assert full == want[0]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_gloo(world):
    import multiprocessing as mp
    import socket

    import oracle

    rng = np.random.default_rng(world)
    text = rng.integers(0, 2, 5000, dtype=np.uint8).tobytes()
    pats = [text[100:104], text[2500:2540], b"\x00" * 3, b"\x01" * 11, text[4990:5000]]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, text, pats, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    by_rank = {o[0][0]: o for o in outs}
    for k, p in enumerate(pats):
        want = oracle.search(p, text).tolist()
        merged, offs = [], []
        for r in range(world):
            rank, off, total, local = by_rank[r][k]
            assert total == len(want)
            assert off == len(merged)
            merged += local
        assert merged == want


def test_harness_mirror_matches_reference_streams():
    import hashlib
    import json

    from paper_1012_2547_b200 import harness
    from paper_1012_2547_b200.inputs import ROOT_SEED, derive_seed

    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
    cfg1 = harness.generate_rand_text(4, 1 << 20, derive_seed(ROOT_SEED, "cfg1", "text"))
    assert hashlib.sha1(cfg1.data).hexdigest()[:16] == fx["cfg1"]["text"]
    (p,) = harness.sample_patterns(cfg1, 8, 1, derive_seed(ROOT_SEED, "cfg1", "pat"))
    assert p.data.hex() == fx["cfg1"]["pattern"]
    assert harness.state_word_count(64) == 1 and harness.state_word_count(65) == 2
    with pytest.raises(ValueError):
        harness.generate_rand_text(3, 10, 1)
    with pytest.raises(ValueError):
        harness.BenchConfig(lengths=(4, 2))
    with pytest.raises(ValueError):
        harness.run_benchmark(harness.BenchConfig(metric="reads"), [cfg1])
