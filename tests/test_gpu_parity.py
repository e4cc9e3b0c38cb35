"""GPU parity: the sm_100a engine (through the C ABI) vs the CPU oracle.

Bit-exact on every position (integer work: no tolerance).  Cases follow the
reference suite's generators (tests/cases.py) plus GPU-specific edges: tile
and halo boundaries, misaligned text pointers, dense/periodic matches,
capacity overflow and batched CSR output.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_1012_2547_b200 as mb
from cases import KNOWN, fuzz_cases, rand_bytes
from paper_1012_2547_b200 import engine

pytestmark = pytest.mark.gpu
TILE = 16384  # boundary spacing of the plants (the engine's tiles are 32 KiB: 2 of these)
ENGINE_TILE = 32768
SEG = 2048


def gpu_positions(p: bytes, t, family="auto") -> np.ndarray:
    plan = engine.Plan(p, family)
    return engine.find(plan, t).cpu().numpy()


def check(p: bytes, t: bytes, family="auto"):
    want = oracle.search(p, t)
    got = gpu_positions(p, t, family) if len(p) <= len(t) else np.empty(0, np.int64)
    assert np.array_equal(got, want), (
        f"m={len(p)} n={len(t)} fam={family}: got {got[:8]} (#{got.size}) want {want[:8]} (#{want.size})")


def test_known_answers(cuda):
    for p, t, exp in KNOWN:
        assert mb.brute_force_search(p, t) == exp
        assert mb.search_hor(p, t) == exp


def test_entry_points_agree(cuda):
    t = b"abracadabra" * 50
    p = b"abra"
    exp = oracle.search(p, t).tolist()
    for fn in (mb.search_hor, mb.search_qs, mb.search_br, mb.search_tvsbs, mb.search_fjs, mb.search_bom,
               mb.search_ebom, mb.search_so, mb.search_sa, mb.search_bndm, mb.search_sbndm, mb.search_lbndm,
               mb.search_sbndm_bmh, mb.search_bmh_sbndm, mb.search_fsbndm):
        assert fn(p, t) == exp, fn.__name__
    assert mb.search_hashq(3, p, t) == exp
    assert mb.search_sbndmq(4, p, t) == exp
    assert mb.get_algorithm("B200").search(p, t) == exp


@pytest.mark.parametrize("lo,hi,n_max,count", [
    (1, 3, 600, 300), (4, 6, 600, 300), (7, 16, 1200, 300), (17, 64, 2048, 300),
    (65, 300, 4096, 200), (301, 1024, 8192, 120), (1025, 4096, 12000, 40),
])
def test_fuzz_vs_oracle(cuda, lo, hi, n_max, count):
    for p, t in fuzz_cases(1000 + lo, count, lo, hi, n_max=n_max):
        check(p, t)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8, 15, 16, 17, 31, 32, 33, 63, 64, 100, 128, 500, 1024])
def test_tile_boundaries(cuda, m):
    rng = np.random.default_rng(m)
    n = 3 * TILE + 1000
    t = bytearray(rand_bytes(rng, 256, n))
    p = rand_bytes(rng, 256, m)
    plants = []
    for b in (TILE, 2 * TILE, 3 * TILE):
        for d in (-m - 3, -m, -m + 1, -5, -1, 0, 1, 3, 7):
            s = b + d
            if 0 <= s <= n - m:
                plants.append(s)
    plants += [0, n - m]
    for s in sorted(set(plants)):
        t[s : s + m] = p
    check(p, bytes(t))


@pytest.mark.parametrize("off", list(range(16)))
def test_misaligned_text(cuda, off):
    rng = np.random.default_rng(100 + off)
    base = torch.from_numpy(np.frombuffer(rand_bytes(rng, 4, 70000 + 64), dtype=np.uint8).copy()).cuda()
    n = 70000 - off
    view = base[off : off + n]
    host = view.cpu().numpy().tobytes()
    for m in (1, 2, 3, 5, 8, 13, 40):
        i = int(rng.integers(0, n - m + 1))
        p = host[i : i + m]
        got = gpu_positions(p, view)
        assert np.array_equal(got, oracle.search(p, host)), (off, m)


@pytest.mark.parametrize("m", [2, 3, 5, 16, 17, 64, 128, 1024, 2000])
def test_dense_periodic(cuda, m):
    rng = np.random.default_rng(m)
    n = 5 * TILE + 123
    t = np.full(n, ord("a"), dtype=np.uint8)
    noise = rng.choice(n, size=n // 1000, replace=False)
    t[noise] = rng.integers(ord("b"), ord("z") + 1, size=noise.size, dtype=np.uint8)
    tb = t.tobytes()
    check(b"a" * m, tb)
    check(b"a" * (m - 1) + b"b", tb)
    check((b"ab" * m)[:m], (b"ab" * n)[:n])
    check((b"abc" * m)[:m], (b"abc" * n)[:n] )
    check(b"a" * m, b"a" * n)


def test_sigma1_and_zero_bytes(cuda):
    for m in (1, 2, 4, 7, 32, 100):
        check(b"\x00" * m, b"\x00" * 3000)
        check(b"\x00" * m, b"\x00" * 3000 + b"\x01" + b"\x00" * 50)


@pytest.mark.parametrize("family,lo,hi", [("win4", 4, 40), ("aligned", 7, 200), ("shiftor", 1, 64), ("swar", 5, 8),
                                          ("gram", 15, 300)])
def test_forced_families(cuda, family, lo, hi):
    for p, t in fuzz_cases(77, 150, lo, hi, n_max=3000):
        check(p, t, family)


@pytest.mark.parametrize("sigmas", [(256,), (64, 128), (8, 16), (2, 4)])
def test_sampled_family(cuda, sigmas):
    """K3 sampled q-gram filter: whenever a plan picks it, results equal the oracle."""
    used = 0
    for p, t in fuzz_cases(500 + sigmas[0], 120, 272, 3000, sigmas=sigmas, n_max=60000):
        try:
            engine.Plan(p, "sampled")
        except ValueError:
            continue  # low entropy / periodic: the plan keeps the full scan
        used += 1
        check(p, t, "sampled")
        check(p, t)
    if sigmas[0] >= 8:
        assert used > 50


def test_sampled_plants_and_edges(cuda):
    rng = np.random.default_rng(7)
    assert engine.Plan(rand_bytes(rng, 256, 272)).info().family != "sampled"  # period below K3_MIN_PERIOD
    for m in (300, 1024, 2047, 4096):
        p = rand_bytes(rng, 256, m)
        assert engine.Plan(p).info().family == "sampled"
        n = 3 * TILE + 4321
        t = bytearray(rand_bytes(rng, 256, n))
        for s in (0, 1, 15, 16, TILE - m, TILE - 1, TILE, 2 * TILE - 7, n - m - 1, n - m):
            if 0 <= s <= n - m:
                t[s : s + m] = p
        check(p, bytes(t))
        base = torch.from_numpy(np.frombuffer(bytes(t) + b"\0" * 32, dtype=np.uint8).copy()).cuda()
        for off in (1, 7, 13):
            view = base[off : off + n - off]
            got = gpu_positions(p, view)
            assert np.array_equal(got, oracle.search(p, bytes(t)[off:n])), (m, off)


@pytest.mark.parametrize("period", [60, 150, 294, 300, 520])
def test_sampled_dense_periodic_occurrences(cuda, period):
    """Long patterns with a short period over texts that repeat it: up to one
    occurrence every `period` bytes.  The planner keeps the sampled family only
    when a unit's occurrences fit its lists (period >= K3_MIN_PERIOD = 294);
    either way every position must come out."""
    rng = np.random.default_rng(period)
    unit = rand_bytes(rng, 256, period)
    p = (unit * (1 + 1100 // period))[:1024]
    t = rand_bytes(rng, 256, 3000) + unit * ((6 << 20) // period) + rand_bytes(rng, 256, 3000)
    fam = engine.Plan(p).info().family
    if period < 294:
        assert fam != "sampled", fam
    check(p, t)


@pytest.mark.parametrize("m", [1, 7, 31, 32, 33, 63, 64])
def test_shiftor_edges(cuda, m):
    rng = np.random.default_rng(300 + m)
    for sigma in (1, 2, 4, 256):
        n = 2 * TILE + 777
        t = bytearray(rand_bytes(rng, sigma, n))
        p = rand_bytes(rng, sigma, m)
        for s in (0, 5, TILE - m, TILE - 1, TILE, n - m):
            t[s : s + m] = p
        check(p, bytes(t), "shiftor")
        base = torch.from_numpy(np.frombuffer(bytes(t) + b"\0" * 32, dtype=np.uint8).copy()).cuda()
        for off in (3, 9):
            got = engine.find(engine.Plan(p, "shiftor"), base[off:n]).cpu().numpy()
            assert np.array_equal(got, oracle.search(p, bytes(t)[off:n])), (m, sigma, off)


def test_shiftor_foreign_bytes_and_code_collisions(cuda):
    """K2 packs text bytes into 1-2 symbol bit planes chosen for the pattern's
    alphabet: bytes outside it alias to a pattern symbol's code (candidates the
    verification must reject), and alphabets no two byte bits can separate
    ({0,1,2,4}) share codes."""
    rng = np.random.default_rng(4242)
    n = 3 * ENGINE_TILE + 1234
    for sym, noise in (([0x41, 0x43], [0x45, 0x47, 0x61, 0x63, 0xC1]),       # A/C differ in bit 1 only
                       ([0, 1, 2, 4], [8, 16, 3, 5, 6, 255]),               # no separating bit pair
                       ([0x41, 0x43, 0x47, 0x54], [0x4E, 0x61, 0x63, 0x00]),  # ACGT + N / lower case
                       ([7, 7 ^ 0x80], [0x07 ^ 0x01, 0x87 ^ 0x10])):
        for m in (1, 2, 5, 8, 13, 31, 32, 33, 64):
            syms = np.array(sym, dtype=np.uint8)
            t = syms[rng.integers(0, len(sym), n)]
            # a tenth of the text replaced by bytes that alias onto pattern codes
            idx = rng.choice(n, n // 10, replace=False)
            t[idx] = np.array(noise, dtype=np.uint8)[rng.integers(0, len(noise), idx.size)]
            p = bytes(syms[rng.integers(0, len(sym), m)])
            tb = bytearray(t.tobytes())
            for s0 in (0, SEG - 3, ENGINE_TILE - m, ENGINE_TILE - 1, 2 * ENGINE_TILE - m // 2, n - m):
                tb[s0 : s0 + m] = p
            check(p, bytes(tb), "shiftor")


@pytest.mark.parametrize("sigma", [2, 3, 4, 8])
def test_shiftor_auto_small_alphabets(cuda, sigma):
    """Auto plans over small alphabets at 5 <= m <= 64 (K2 where the word filters
    are busy) equal the oracle; sigma = 2, m = 8 must take K2."""
    rng = np.random.default_rng(900 + sigma)
    n = 4 * ENGINE_TILE + 999
    t = rand_bytes(rng, sigma, n)
    fams = set()
    for m in (5, 6, 7, 8, 9, 12, 14, 16, 20, 22, 24, 33, 48, 64):
        off = int(rng.integers(0, n - m))
        p = t[off : off + m]
        fams.add((m, engine.Plan(p).info().family))
        check(p, t)
    if sigma == 2:
        assert (8, "shiftor") in fams, fams


@pytest.mark.parametrize("m", [7, 9, 15, 16, 33, 64, 200, 1000])
def test_run_filter_edges_and_capacity(cuda, m):
    """c^m (the exact run filter, m >= 7) on a text larger than one resident
    wave (the 3-launch pipeline: run-table and staged expansion), runs of c
    ending and starting at tile and segment boundaries and at the text edges,
    every pointer misalignment, and an output buffer cut inside a dense
    segment (prefix of the list, full count)."""
    n = 12 << 20  # > the fused single-wave limit
    t = np.zeros(n, dtype=np.uint8) + ord("q")
    rng = np.random.default_rng(60 + m)
    t[rng.choice(n, n // 3000, replace=False)] = ord("z")  # long runs broken by rare bytes
    for b in (ENGINE_TILE, 7 * ENGINE_TILE, 5 * SEG, 100 * SEG + 3):
        for d in (-m - 1, -m, -m + 1, -1, 0, 1):
            t[b + d] = ord("z")
    t[:3] = ord("z")
    t[n - m - 2] = ord("z")
    t[200 * SEG : 260 * SEG : 2] = ord("z")  # every other byte: no match, dozens of 1-byte runs per segment
    t[300 * SEG : 330 * SEG] = np.frombuffer(b"qqqz" * (30 * SEG // 4), dtype=np.uint8)  # runs of 3
    p = b"q" * m
    assert engine.Plan(p).info().period == 1
    base = torch.from_numpy(np.concatenate([np.zeros(16, np.uint8), t])).cuda()
    host = t.tobytes()
    want = oracle.search(p, host, threads=4)
    for off in (0, 1, 7, 15):
        view = base[16 - off : 16 - off + n + off][off:] if off else base[16 : 16 + n]
        got = engine.find(engine.Plan(p), view).cpu().numpy()
        assert np.array_equal(got, want), (m, off, got.size, want.size)
    # capacity cut inside a dense segment
    cap = int(want.size // 2 + 777)
    out = torch.full((cap + 8,), -1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    engine.find_into(engine.Plan(p), base[16 : 16 + n], out[:cap], cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == want.size
    assert np.array_equal(out[:cap].cpu().numpy(), want[:cap])
    assert (out[cap:] == -1).all(), "wrote past the capacity"


@pytest.mark.parametrize("sigma", [2, 3, 4, 16, 256])
def test_plans_with_text_histogram(cuda, sigma):
    """Plans built with the text's byte histogram (K0 on the device, the text side
    of the reference's select(pattern, text)): anchors, bit planes and families are
    chosen from the true byte probabilities -- results equal the oracle for every
    m, and the families are the small-alphabet ones where they should be."""
    rng = np.random.default_rng(8100 + sigma)
    n = 5 * ENGINE_TILE + 321
    t = rand_bytes(rng, sigma, n)
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    hist = engine.histogram(d).cpu().numpy()
    assert int(hist.sum()) == n and int((hist > 0).sum()) <= sigma
    fams = {}
    for m in (1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 15, 16, 23, 31, 40, 64, 65, 300):
        off = int(rng.integers(0, n - m))
        p = t[off : off + m]
        pl = engine.Plan(p, hist=hist)
        fams[m] = pl.info().family
        got = engine.find(pl, d).cpu().numpy()
        assert np.array_equal(got, oracle.search(p, t)), (sigma, m, fams[m])
    if sigma == 4:
        assert fams[5] == fams[6] == "swar", fams
    if sigma == 256:
        assert fams[5] == "win4" and fams[8] == "aligned", fams


@pytest.mark.parametrize("tiles", [1, 2, 150, 295, 296, 297, 300, 450])
def test_single_wave_fused_boundary(cuda, tiles):
    """Texts of up to one resident wave of tiles run as ONE fused launch (scan,
    look-back over tiles, positions written directly); one tile more takes the
    scan / offsets / expand pipeline.  Both must agree with the oracle, for
    sparse, dense (sigma = 2, m = 3), periodic and long patterns, and for the
    last alignment of the text."""
    rng = np.random.default_rng(4000 + tiles)
    n = tiles * ENGINE_TILE - 37
    t = bytearray(rand_bytes(rng, 2, n))
    pats = [bytes(t[5:8]), bytes(t[n - 40 : n - 20]), b"\x00\x01" * 40, bytes(t[n - 300 :])]
    for p in pats:
        check(p, bytes(t))
    p = bytes(t[1000:1003])
    want = oracle.search(p, bytes(t))
    plan = engine.Plan(p)
    d = torch.from_numpy(np.frombuffer(bytes(t), dtype=np.uint8).copy()).cuda()
    out = torch.empty(want.size + 1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    l0 = engine.launch_count()
    engine.find_into(plan, d, out, cnt)
    launches = engine.launch_count() - l0
    assert int(cnt.item()) == want.size
    assert np.array_equal(out[: want.size].cpu().numpy(), want)
    # one wave: >= 2 resident CTAs per SM x 148 SMs, at most 3 (544-thread CTAs)
    if tiles <= 296:
        assert launches == 1, launches
    elif tiles > 3 * 148:
        assert launches == 3, launches
    else:
        assert launches in (1, 3), launches


def test_single_wave_dense_and_capacity(cuda):
    """Fused single-wave search with every position a match (sigma = 1), count
    only, and a capacity cut in the middle of a tile."""
    t = b"a" * (4 << 20)
    for m in (1, 2, 9, 64, 700):
        check(b"a" * m, t)
    plan = engine.Plan(b"aaa")
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    assert engine.count(plan, d) == len(t) - 2
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.full((50000,), -1, dtype=torch.int64, device="cuda")
    engine.find_into(plan, d, out, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == len(t) - 2
    assert np.array_equal(out.cpu().numpy(), np.arange(50000))


def test_count_only_and_overflow(cuda):
    rng = np.random.default_rng(5)
    t = rand_bytes(rng, 2, 200000)
    p = t[100:104]
    want = oracle.search(p, t)
    plan = engine.Plan(p)
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    assert engine.count(plan, d) == want.size
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.full((100,), -1, dtype=torch.int64, device="cuda")
    engine.find_into(plan, d, out, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == want.size
    assert np.array_equal(out.cpu().numpy(), want[:100])


def test_batch_csr(cuda):
    rng = np.random.default_rng(9)
    t = rand_bytes(rng, 8, 300000)
    pats = [t[i : i + m] for i, m in zip(rng.integers(0, 290000, 40), rng.integers(1, 300, 40))]
    pats += [b"\x07\x07", b"\x01" * 9, b"zzz" * 50]
    res = mb.search_many(pats, t)
    for p, r in zip(pats, res):
        assert r == oracle.search(p, t).tolist()


def test_host_entry(cuda):
    rng = np.random.default_rng(11)
    t = np.frombuffer(rand_bytes(rng, 4, 100000), dtype=np.uint8)
    for m in (3, 9, 70):
        p = t[500 : 500 + m].tobytes()
        assert np.array_equal(engine.search_host(p, t, cap=4), oracle.search(p, t))


def test_histogram_alphabet(cuda):
    rng = np.random.default_rng(12)
    t = rand_bytes(rng, 37, 100000)
    h = engine.histogram(t).cpu().numpy()
    assert np.array_equal(h, np.bincount(np.frombuffer(t, np.uint8), minlength=256))
    assert mb.Text(t).alphabet_size() == len(set(t))
    # K0 reads 16-byte vectors: every pointer misalignment, lengths around the vector and
    # block sizes, a text of one byte value (every lane on one bin), a multi-block text
    base = torch.from_numpy(np.frombuffer(rand_bytes(rng, 256, (9 << 20) + 64), np.uint8).copy()).cuda()
    hb = base.cpu().numpy()
    for off in (0, 1, 7, 15):
        for n in (0, 1, 15, 16, 17, 31, 4097, 65536 + 5, (9 << 20) + 3):
            got = engine.histogram(base[off : off + n]).cpu().numpy()
            assert np.array_equal(got, np.bincount(hb[off : off + n], minlength=256)), (off, n)
    ones = torch.full((3 << 20,), 7, dtype=torch.uint8, device="cuda")
    h1 = engine.histogram(ones[3:]).cpu().numpy()
    assert h1[7] == (3 << 20) - 3 and h1.sum() == h1[7]


def test_instrumented_text_rejected(cuda):
    with pytest.raises(TypeError):
        mb.search_hor(b"ab", mb.InstrumentedText(b"abab"))


@pytest.mark.parametrize("sigma,m", [(16, 8), (64, 16), (256, 9), (95, 40), (32, 200)])
def test_mp_batched_single_pass(cuda, sigma, m):
    """K5 multi-pattern pass (selective ALIGNED batches): CSR equals per-pattern oracle results,
    including duplicate patterns, planted repeats and patterns longer than the text."""
    rng = np.random.default_rng(sigma * 1000 + m)
    n = 3 * TILE + 4099
    t = bytearray(rand_bytes(rng, sigma, n))
    pats = [bytes(t[i : i + m]) for i in rng.integers(0, n - m, 300)]
    pats += [pats[0], pats[1], rand_bytes(rng, sigma, m)]
    for s in (0, 7, TILE - 3, n - m):  # plant pattern 2 at edges / tile boundary
        t[s : s + m] = pats[2]
    t = bytes(t)
    before = engine.mp_batches()
    res = mb.search_many(pats, t)
    assert engine.mp_batches() == before + 1, "selective ALIGNED batch did not take the MP pass"
    for p, r in zip(pats, res):
        assert r == oracle.search(p, t).tolist(), (len(p), p[:4])


def test_mp_mixed_family_batch(cuda):
    """K5 pass over a batch mixing families (ALIGNED 1/2 words, WIN4, shift-or,
    sampled with deltas up to S-1 > one segment): every hit lands in its own
    family's bitmap coordinates, so the CSR equals the oracle per pattern."""
    rng = np.random.default_rng(2718)
    n = 5 * TILE + 123
    t = bytearray(rand_bytes(rng, 256, n))
    specs = [(24, "auto", 0)] * 100 + [(24, "win4", 0)] * 40 + [(40, "shiftor", 0)] * 20 + \
            [(64, "auto", 2)] * 10 + [(int(m), "auto", 0) for m in rng.integers(300, 1500, 30)]
    pats, plans = [], []
    for m, fam, nw in specs:
        i = int(rng.integers(0, n - m))
        p = bytes(t[i : i + m])
        pats.append(p)
        plans.append(engine.Plan(p, fam, anchor_words=nw))
    for s in (0, SEG - 5, TILE - 3, n - len(pats[-1])):  # plant a sampled-family pattern at edges
        t[s : s + len(pats[-1])] = pats[-1]
    t = bytes(t)
    fams = {pl.info().family for pl in plans}
    assert {"aligned", "win4", "shiftor", "sampled"} <= fams, fams
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    for obj in (plans, engine.Batch(plans)):
        before = engine.mp_batches()
        pos, offs = engine.find_batch(obj, d)
        assert engine.mp_batches() == before + 1, "mixed batch did not take the MP pass"
        pos = pos.cpu().numpy()
        for k, p in enumerate(pats):
            assert np.array_equal(pos[offs[k] : offs[k + 1]], oracle.search(p, t)), (k, len(p))


@pytest.mark.parametrize("sigma,lo,hi", [(16, 2, 3), (64, 4, 6), (256, 2, 9), (4, 8, 20), (8, 5, 40), (32, 3, 300),
                                         (2, 16, 64), (2, 20, 300)])
def test_mpb_byte_offset_pass(cuda, sigma, lo, hi):
    """K5b byte-offset pass (short patterns / small alphabets): planted edges,
    duplicates, patterns longer than the text; ad-hoc and prepared batches."""
    rng = np.random.default_rng(sigma * 100 + lo)
    n = 3 * TILE + 777
    t = bytearray(rand_bytes(rng, sigma, n))
    ms = rng.integers(lo, hi + 1, 240)
    pats = [bytes(t[i : i + m]) for i, m in zip(rng.integers(0, n - hi, 240), ms)]
    pats += [pats[0], rand_bytes(rng, sigma, lo), rand_bytes(rng, sigma, hi)]
    for s in (0, 1, SEG - 1, TILE - 2, n - len(pats[3])):
        t[s : s + len(pats[3])] = pats[3]
    t = bytes(t)
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    plans = [engine.Plan(p) for p in pats]
    for obj in (plans, engine.Batch(plans)):
        before = engine.mp_batches()
        pos, offs = engine.find_batch(obj, d)
        assert engine.mp_batches() == before + 1, "batch did not take a batched pass"
        pos = pos.cpu().numpy()
        for k, p in enumerate(pats):
            assert np.array_equal(pos[offs[k] : offs[k + 1]], oracle.search(p, t)), (k, p)


def test_batch_with_every_family_group(cuda):
    """One batch spanning ten family keys (SWAR m=1/2/3, WIN4, ALIGNED
    1/2/3 words, sampled, K2 with one and two bit planes): one count launch per group."""
    rng = np.random.default_rng(404)
    n = 2 * TILE + 999
    t = rand_bytes(rng, 256, n)
    tb = rand_bytes(rng, 2, 4096)
    t = t[:9000] + tb + t[9000 + len(tb):]
    specs = [(t[100:101], "auto", 0), (t[200:202], "auto", 0), (t[300:303], "auto", 0), (t[400:405], "auto", 0),
             (t[500:524], "auto", 1), (tb[10:50], "auto", 2), (tb[100:160], "auto", 3),
             (t[700:1300], "auto", 0), (tb[2000:2020], "shiftor", 0), (t[3000:3050], "shiftor", 0)]
    plans = [engine.Plan(p, fam, anchor_words=nw) for p, fam, nw in specs]
    keys = {(pl.info().family, pl.m if pl.info().family == "swar" else pl.info().words) for pl in plans}
    assert len(keys) == 10, keys
    for obj in (plans, plans * 3):
        pos, offs = engine.find_batch(obj, t)
        pos = pos.cpu().numpy()
        for k, pl in enumerate(obj):
            assert np.array_equal(pos[offs[k] : offs[k + 1]], oracle.search(pl.pattern, t)), (k, pl.m)


@pytest.mark.parametrize("n", [0, 1, 5, 100, 3000])
def test_batched_passes_tiny_texts(cuda, n):
    """Batched passes (and their fallbacks) on texts shorter than many of the
    patterns, down to the empty text."""
    rng = np.random.default_rng(n + 17)
    for sigma in (4, 64, 256):
        t = rand_bytes(rng, sigma, n)
        pats = [rand_bytes(rng, sigma, int(m)) for m in rng.integers(1, 40, 30)]
        pats += [t[i : i + 3] for i in range(0, max(n - 3, 0), max(n // 7, 1))][:10]
        pats = [p for p in pats if p]
        for obj in (None, "prepared"):
            plans = [engine.Plan(p) for p in pats]
            pos, offs = engine.find_batch(engine.Batch(plans) if obj else plans, t)
            pos = pos.cpu().numpy()
            for k, p in enumerate(pats):
                want = oracle.search(p, t) if len(p) <= n else np.empty(0, np.int64)
                assert np.array_equal(pos[offs[k] : offs[k + 1]], want), (sigma, k, len(p), n)


def test_mpb_overflow_falls_back(cuda):
    # selective-looking short patterns, but one of them repeats > LIST_CAP times in a segment
    rng = np.random.default_rng(77)
    t = bytearray(rand_bytes(rng, 64, 2 * TILE))
    t[5000:5400] = b"xy" * 200
    t = bytes(t)
    pats = [t[i : i + 2] for i in rng.integers(0, len(t) - 2, 40)] + [b"xy", b"yx"]
    res = mb.search_many(pats, t)
    for p, r in zip(pats, res):
        assert r == oracle.search(p, t).tolist()


def test_prepared_batch_matches_adhoc(cuda):
    rng = np.random.default_rng(44)
    t = rand_bytes(rng, 128, 4 * TILE)
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    pats = [t[i : i + 24] for i in rng.integers(0, len(t) - 24, 700)] + [t[5:9], t[100:2100]]
    plans = [engine.Plan(p) for p in pats]
    batch = engine.Batch(plans)
    before = engine.mp_batches()
    pos_b, offs_b = engine.find_batch(batch, d)
    pos_a, offs_a = engine.find_batch(plans, d)
    assert torch.equal(pos_a, pos_b) and torch.equal(offs_a, offs_b)
    for k in (0, 1, 500, 700, 701):
        assert pos_b[offs_b[k] : offs_b[k + 1]].cpu().tolist() == oracle.search(pats[k], t).tolist()
    mp = engine.Batch([engine.Plan(p) for p in pats[:600]])  # all ALIGNED: prepared MP tables (2 chunks)
    pos_m, offs_m = engine.find_batch(mp, d)
    assert engine.mp_batches() >= before + 1
    assert torch.equal(pos_m, pos_a[: int(offs_a[600])]) and torch.equal(offs_m, offs_a[:601])


def test_mp_overflow_falls_back(cuda):
    # a dense, selective-looking batch: every pattern occurs > LIST_CAP times per 2 KiB segment
    rng = np.random.default_rng(5)
    unit = rand_bytes(rng, 256, 40)
    t = unit * 4000
    pats = [unit[i:] + unit[:i] for i in range(16)]
    res = mb.search_many(pats, t)
    for p, r in zip(pats, res):
        assert r == oracle.search(p, t).tolist()


def test_mp_overflow_with_duplicates(cuda):
    """Duplicates of patterns whose batch-pass segments overflow: the
    representative falls back to its family scan and every copy still reads
    the representative's (rescanned) segments."""
    rng = np.random.default_rng(6)
    unit = rand_bytes(rng, 256, 40)
    t = rand_bytes(rng, 256, 50_000) + unit * 4000 + rand_bytes(rng, 256, 50_000)
    dense = [unit[i:] + unit[:i] for i in range(8)]
    sparse = [t[i : i + 24] for i in rng.integers(0, 50_000, 24)]
    pats = dense + sparse + dense[::-1] + sparse[:5] + dense[:3]
    res = mb.search_many(pats, t)
    for p, r in zip(pats, res):
        assert r == oracle.search(p, t).tolist()


def test_compiled_searcher_shared_across_threads(cuda):
    """tests/test_registry.py:152-162 analog: one compiled run(hay) used from 4 threads."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(99)
    t = rand_bytes(rng, 4, 20000)
    p = t[1234:1246]
    expected = oracle.search(p, t).tolist()
    for algo_id in ("HOR", "EBOM", "SBNDM", "HASH5", "B200"):
        run = mb.get_algorithm(algo_id).compile(p)
        with ThreadPoolExecutor(max_workers=4) as pool:
            results = list(pool.map(run, [t] * 16))
        assert all(r == expected for r in results), algo_id


def test_streams_and_device_tensor_inputs(cuda):
    rng = np.random.default_rng(7)
    t = rand_bytes(rng, 256, 3 * TILE)
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    p = t[500:540]
    plan = engine.Plan(p)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        got = engine.find(plan, d, stream=s)
    s.synchronize()
    assert got.cpu().tolist() == oracle.search(p, t).tolist()
    run = mb.compile_tensor(p)
    assert run(d).cpu().tolist() == oracle.search(p, t).tolist()


def test_one_context_two_streams_unsynchronised(cuda):
    """Searches of one context (one thread) issued back to back on two streams
    without synchronisation: the engine orders them (they share the context's
    tickets and scratch), so both results are complete."""
    rng = np.random.default_rng(8)
    t = rand_bytes(rng, 4, 24 << 20)
    d = torch.from_numpy(np.frombuffer(t, dtype=np.uint8).copy()).cuda()
    pats = [t[1000:1006], t[5000:5009], b"\x00\x01\x02", t[7 << 20 : (7 << 20) + 40]]
    plans = [engine.Plan(p) for p in pats]
    wants = [oracle.search(p, t) for p in pats]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty(w.size + 1, dtype=torch.int64, device="cuda") for w in wants]
    cnts = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in wants]
    torch.cuda.synchronize()
    for i, (pl, o, c) in enumerate(zip(plans, outs, cnts)):
        engine.find_into(pl, d, o, c, streams[i % 2])
    torch.cuda.synchronize()
    for w, o, c in zip(wants, outs, cnts):
        assert int(c.item()) == w.size
        assert np.array_equal(o[: w.size].cpu().numpy(), w)


def test_batch_sub_batching_chains_csr(cuda, monkeypatch):
    """A batch larger than the scratch budget runs as chained sub-batches (MP and
    per-pattern paths, patterns longer than the text included)."""
    rng = np.random.default_rng(31)
    t = rand_bytes(rng, 64, 6000)
    pats = [t[i : i + m] for i, m in zip(rng.integers(0, len(t) - 300, 60), rng.integers(7, 300, 60))]
    pats += [b"\x05" * 7000, t[:3], t[10:15]]
    want = [oracle.search(p, t).tolist() for p in pats]
    monkeypatch.setenv("MB_SCRATCH_BUDGET", str(200_000))  # a few patterns per sub-batch
    assert mb.search_many(pats, t) == want
    monkeypatch.setenv("MB_SCRATCH_BUDGET", str(1))  # one pattern per sub-batch
    assert mb.search_many(pats, t) == want


@pytest.mark.parametrize("sigma,m", [(2, 2), (2, 8), (4, 4), (64, 16), (4, 300)])
def test_batch_duplicate_patterns(cuda, sigma, m, monkeypatch):
    """Identical patterns of a batch are searched once and their CSR ranges
    filled from the representative's segments: every copy must still get the
    complete list, through the batch passes, the per-pattern scans and chained
    sub-batches (where a copy's representative may sit in an earlier one)."""
    rng = np.random.default_rng(7000 + sigma + m)
    t = rand_bytes(rng, sigma, 300_000)
    base = [t[i : i + m] for i in rng.integers(0, len(t) - m, 12)]
    pats = [base[i] for i in rng.integers(0, len(base), 120)] + [b"\x00" * (m + 1), base[0]]
    want = {p: oracle.search(p, t).tolist() for p in set(pats)}
    res = mb.search_many(pats, t)
    assert [len(r) for r in res] == [len(want[p]) for p in pats]
    assert all(r == want[p] for r, p in zip(res, pats))
    monkeypatch.setenv("MB_SCRATCH_BUDGET", str(3_000_000))  # sub-batches of a few patterns
    res = mb.search_many(pats, t)
    assert all(r == want[p] for r, p in zip(res, pats))


def test_batch_every_family_key_with_pass(cuda):
    """All 16 family keys of engine.cu family_key (SWAR m = 1,2,3,5..8, WIN4,
    even-window WIN4, ALIGNED 1/2/3 words, the c^m run filter, sampled,
    K2 with one / two bit planes) in ONE batch together with enough sparse long patterns for
    a batch pass -- every key then launches twice (ungated, and gated behind
    the pass's overflow flag): 32 count-kernel groups, the ticket-slot limit."""
    rng = np.random.default_rng(405)
    n = 6 * ENGINE_TILE + 777
    t = bytearray(rand_bytes(rng, 256, n))
    tb = rand_bytes(rng, 2, 8192)
    t[20000:20000 + len(tb)] = tb
    t[40000:40300] = b"\x07" * 300
    t = bytes(t)
    specs = [(t[100:101], "auto", 0), (t[200:202], "auto", 0), (t[300:303], "auto", 0),
             (t[400:404], "auto", 0), (t[450:455], "auto", 0)]
    specs += [(tb[i * 40: i * 40 + m], "swar", 0) for i, m in enumerate((5, 6, 7, 8), 1)]
    specs += [(t[500:524], "auto", 1), (tb[300:340], "auto", 2), (tb[400:460], "auto", 3),
              (b"\x07" * 20, "auto", 0), (t[60000:60700], "auto", 0),
              (tb[2000:2020], "shiftor", 0), (t[3000:3050], "shiftor", 0)]
    plans = [engine.Plan(p, fam, anchor_words=nw) for p, fam, nw in specs]
    infos = [pl.info() for pl in plans]
    keys = {(i.family, i.m if i.family == "swar" else i.words,
             i.periodic and i.period == 1 if i.family == "aligned" else i.m == 4 if i.family == "win4" else None)
            for i in infos}
    assert len(keys) == 16, keys
    # sparse m >= 7 patterns for the aligned-word batch pass (the short ones make it byte-offset)
    sparse = [t[i : i + 32] for i in rng.integers(70000, n - 40, 40)]
    mp0 = engine.mp_batches()
    for obj in (plans + [engine.Plan(p) for p in sparse], [engine.Plan(p) for p in sparse] + plans * 2):
        for b in (obj, engine.Batch(obj)):
            pos, offs = engine.find_batch(b, t)
            pos = pos.cpu().numpy()
            for k, pl in enumerate(obj):
                assert np.array_equal(pos[offs[k] : offs[k + 1]], oracle.search(pl.pattern, t)), (k, pl.m)
    assert engine.mp_batches() > mp0, "no batch pass: the gated groups were not exercised"


@pytest.mark.parametrize("sigma", [2, 4, 8])
def test_gram_family_small_alphabets(cuda, sigma):
    """K1G strided gram filter (auto for small alphabets at m >= 15..31): every
    (S, Q) variant, occurrences planted across tile and segment boundaries, at
    the text edges, over all 16 pointer misalignments, and dense self-overlapping
    patterns (forced) whose grams hit at every sample."""
    rng = np.random.default_rng(500 + sigma)
    n = 3 * ENGINE_TILE + 999
    variants = set()
    for m in (15, 16, 22, 23, 24, 30, 31, 32, 47, 64, 65, 100, 257):
        t = bytearray(rand_bytes(rng, sigma, n))
        p = bytes(t[777 : 777 + m])
        for b in (ENGINE_TILE, 2 * ENGINE_TILE, SEG * 5):
            for d in (-m - 1, -m + 1, -9, -1, 0, 1, 8, 15):
                if 0 <= b + d <= n - m:
                    t[b + d : b + d + m] = p
        t[:m] = p
        t[n - m :] = p
        t = bytes(t)
        info = engine.Plan(p).info()
        if info.family == "gram":
            variants.add((info.stride, info.gram))
        check(p, t)
        check(p, t, "gram")
    if sigma == 2:
        assert {(8, 16), (16, 16)} <= variants, variants
    if sigma == 4:
        assert {(8, 8), (16, 16)} <= variants, variants
    if sigma == 8:
        assert {(8, 8), (16, 8)} <= variants, variants
    base = torch.from_numpy(np.frombuffer(rand_bytes(rng, sigma, 90000 + 64), dtype=np.uint8).copy()).cuda()
    for off in range(16):
        view = base[off : off + 90000 - off]
        host = view.cpu().numpy().tobytes()
        for m in (15, 23, 31, 40):
            i = int(rng.integers(0, len(host) - m))
            p = host[i : i + m]
            for fam in ("auto", "gram"):
                got = engine.find(engine.Plan(p, fam), view).cpu().numpy()
                assert np.array_equal(got, oracle.search(p, host)), (off, m, fam)
    for unit in (b"ab", b"abc", b"aab", b"abcdefgh"):
        for m in (15, 24, 40, 100):
            p = (unit * 64)[:m]
            t = (unit * (n // len(unit)))[: n - 5] + b"zzzzz"
            check(p, t, "gram")
