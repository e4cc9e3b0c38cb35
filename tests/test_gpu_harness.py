"""GPU: the B200 engine inside the REFERENCE's own harness (SURVEY.md 8(b) "Callers").

The unmodified reference package is installed into baseline/_ref
(tools/install_reference.sh, run by __graft_entry__.build()); these tests import
it from there -- never from /root/reference, which the GPU box does not have --
and hand it the B200 descriptor the way the reference's own tests substitute
algorithms (dataclasses.replace, pkg/tests/test_differential.py:39,72):

* run_differential(10000, seed=2026) -- the acceptance workload
  (pkg/tests/test_acceptance.py:44-54, differential.py:95-131), once with the
  B200 descriptor and once with every registry entry's compile swapped for
  this package's bounded GPU searcher of the same id;
* bench.run_benchmark with the B200 descriptor (bench.py:204-238), counts
  checked against the reference's own HOR run and the C oracle;
* our measurement CSV through report.parse_measurements_csv /
  render_best_map (report.py:138-233), and byte-equal to the reference's
  render_table(..., "csv");
* the reference CLI's `search` (cli.py:139-173) resolving "B200";
* the ctypes binding printed in INTEGRATION.md, executed verbatim.
"""
from __future__ import annotations

import dataclasses
import importlib
import os
import re
import sys

import numpy as np
import pytest

import oracle
import paper_1012_2547_b200 as mb
from paper_1012_2547_b200 import cli, engine
from paper_1012_2547_b200.searchers import compile_engine

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isfile(os.path.join(REF, "matchbench", "__init__.py")):
        pytest.fail("reference package missing: run tools/install_reference.sh (or __graft_entry__.build())")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    m = importlib.import_module("matchbench")
    assert os.path.dirname(m.__file__).startswith(REF), m.__file__
    return m


def b200(ref):
    return dataclasses.replace(ref.get_algorithm("HOR"), id="B200", compile=compile_engine)


def test_reference_run_differential_b200(cuda, ref):
    l0 = engine.launch_count()
    rep = ref.run_differential(10000, seed=2026, algos=[b200(ref)])
    assert rep.total_cases == 10000
    assert rep.ok, "\n".join(x.describe() for x in rep.mismatches[:5])
    assert engine.launch_count() - l0 >= 9000  # the cases ran on the GPU (m > n cases launch nothing)


def test_reference_run_differential_every_entry_point(cuda, ref):
    """The acceptance run over the reference's REGISTRY, each descriptor's
    compile replaced by this package's GPU searcher of the same id (its
    bounds and errors included)."""
    ours = {a.id: a for a in mb.REGISTRY}
    algos = [dataclasses.replace(a, compile=ours[a.id].compile) for a in ref.REGISTRY]
    assert [a.id for a in algos] == [a.id for a in mb.REGISTRY]
    rep = ref.run_differential(10000, seed=2026, algos=algos)
    assert rep.total_cases >= 10000
    assert rep.ok, "\n".join(x.describe() for x in rep.mismatches[:5])


def test_reference_run_benchmark_b200(cuda, ref):
    cfg = ref.BenchConfig(lengths=(2, 8, 32, 128), patterns_per_length=4, text_size=1 << 18, seed=7)
    texts = [ref.generate_rand_text(4, cfg.text_size, 11), ref.generate_rand_text(64, cfg.text_size, 12)]
    ms = ref.run_benchmark(cfg, texts, algos=[b200(ref)])
    base = {(x.text_id, x.m): x for x in ref.run_benchmark(cfg, texts, algos=[ref.get_algorithm("HOR")])}
    assert len(ms) == 8
    for x in ms:
        assert x.algorithm == "B200" and x.metric == "time" and x.mean_value > 0 and x.runs == 4
        assert x.mean_occurrences == base[(x.text_id, x.m)].mean_occurrences
    # the same cells' counts from the C oracle (bench.py:167-201 pattern draw)
    for text in texts:
        t = np.frombuffer(text.data, dtype=np.uint8)
        for m in cfg.lengths:
            pats = ref.sample_patterns(text, m, cfg.patterns_per_length, ref.bench.derive_seed(cfg.seed, text.id, m))
            want = sum(oracle.count(p.data, t) for p in pats) / len(pats)
            got = next(x for x in ms if x.text_id == text.id and x.m == m)
            assert got.mean_occurrences == want


def test_csv_through_reference_report(cuda, ref):
    text = ref.generate_rand_text(8, 1 << 17, 5)
    lengths = (2, 4, 32, 256)
    algos = [mb.get_algorithm("B200"), mb.get_algorithm("SSEF"), mb.get_algorithm("HOR")]
    rows = cli.sort_rows(cli.gpu_benchmark(text.data, text.id, algos, lengths, 3, 9))
    csv_text = cli.render_csv(rows)
    parsed = ref.parse_measurements_csv("# engine=b200\n" + csv_text)
    assert len(parsed) == len(rows)
    t = np.frombuffer(text.data, dtype=np.uint8)
    for r, p in zip(rows, parsed):
        assert (p.text_id, p.sigma, p.family, p.algorithm, p.m, p.metric) == (r[0], r[1], r[2], r[3], r[4], r[8])
        assert p.mean_value == float(cli.format_value(r[5]))
        pats = [t[i : i + r[4]].tobytes() for i in mb.inputs.sample_positions(t.size, r[4], 3,
                                                                                mb.inputs.derive_seed(9, text.id, r[4]))]
        assert r[7] == sum(oracle.count(p, t) for p in pats) / 3  # mean_occurrences vs the oracle
    # byte-equal to the reference's own CSV writer on the same measurements
    as_ref = [ref.Measurement(r[0], r[1], r[2], r[3], r[4], 3, r[5], r[6], r[7], r[8]) for r in rows]
    assert ref.render_table(as_ref, "csv") == csv_text
    best = ref.render_best_map(parsed)
    measured = {(c.sigma_class, c.m_class) for c in (ref.classify(p.sigma, p.m) for p in parsed)}
    for sc, mc in measured:
        cell = best.cell(sc, mc)
        assert cell.algorithm in {"B200", "SSEF", "HOR"} and cell.provenance == "measured"
    assert "| sigma" in best.to_markdown()


def test_reference_cli_search_resolves_b200(cuda, ref, tmp_path, capsys, monkeypatch):
    rcli = importlib.import_module("matchbench.cli")
    orig = rcli.get_algorithm
    monkeypatch.setattr(rcli, "get_algorithm", lambda name: b200(ref) if name == "B200" else orig(name))
    rng = np.random.default_rng(8)
    t = rng.integers(0, 4, 50000, dtype=np.uint8).tobytes()
    f = tmp_path / "t.bin"
    f.write_bytes(t)
    p = t[1234:1242]
    esc = "".join(f"\\x{b:02x}" for b in p)
    assert rcli.main(["search", "--algo", "B200", "--pattern", esc, "--text", str(f)]) == 0
    got = [int(x) for x in capsys.readouterr().out.split()]
    assert got == oracle.search(p, t).tolist()
    assert rcli.main(["search", "--algo", "B200", "--pattern", "\\x09\\x09\\x09", "--text", str(f)]) == 1


def test_integration_md_ctypes_snippet(cuda):
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = next(b for b in re.findall(r"```python\n(.*?)```", md, re.S) if "def compile_b200" in b)
    block = block.replace('ctypes.CDLL("libmatchb200.so")', f"ctypes.CDLL({engine.LIB_PATH!r})")
    ns: dict = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(2)
    t = rng.integers(0, 2, 300000, dtype=np.uint8).tobytes()
    for p in (b"\x00\x01", t[100:109], t[5000:5400]):
        assert ns["compile_b200"](p)(t) == oracle.search(p, t).tolist()
    with pytest.raises(RuntimeError, match="length"):
        ns["compile_b200"](b"")(t)


def test_package_run_differential_and_load_corpus(cuda, tmp_path):
    rep = mb.run_differential(460, seed=5)  # every registry entry, 20 cases each
    assert rep.ok and rep.total_cases == 460
    f = tmp_path / "ecoli"
    f.write_bytes(b"ACGT" * 1000)
    with pytest.warns(UserWarning, match="expected n="):
        txt = mb.load_corpus(f)
    assert txt.id == "ecoli" and len(txt) == 4000 and txt.alphabet_size() == 4
