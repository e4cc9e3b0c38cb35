"""GPU: the CLI behaves like the reference's `matchbench search`
(grep-style exit codes, \\xNN patterns, --algo auto) and writes reference-format CSV rows."""
from __future__ import annotations

import csv
import io

import numpy as np
import pytest

import oracle
from paper_1012_2547_b200 import cli

pytestmark = pytest.mark.gpu


def test_search_exit_codes_and_output(cuda, tmp_path, capsys):
    f = tmp_path / "t.bin"
    f.write_bytes(b"abcabc")
    assert cli.main(["search", "--pattern", "abc", "--text", str(f)]) == 0  # test_cli.py:141-149
    assert capsys.readouterr().out.split() == ["0", "3"]
    assert cli.main(["search", "--pattern", "zzz", "--text", str(f)]) == 1
    assert capsys.readouterr().out == ""
    assert cli.main(["search", "--pattern", "", "--text", str(f)]) == 2
    assert cli.main(["search", "--algo", "SSEF", "--pattern", "ab", "--text", str(f)]) == 2
    assert "m >= 32" in capsys.readouterr().err
    assert cli.main(["search", "--algo", "NOPE", "--pattern", "ab", "--text", str(f)]) == 2


def test_search_escapes_and_auto(cuda, tmp_path, capsys):
    rng = np.random.default_rng(3)
    t = rng.integers(0, 256, 200000, dtype=np.uint8).tobytes()
    f = tmp_path / "r.bin"
    f.write_bytes(t)
    p = t[777:790]
    esc = "".join(f"\\x{b:02x}" for b in p)
    assert cli.main(["search", "--pattern", esc, "--text", str(f)]) == 0
    got = [int(x) for x in capsys.readouterr().out.split()]
    assert got == oracle.search(p, t).tolist()
    assert cli.main(["search", "--pattern", esc, "--text", str(f), "--count"]) == 0
    assert int(capsys.readouterr().out) == len(got)


def test_bench_rows_reference_format(cuda, tmp_path):
    rng = np.random.default_rng(4)
    f = tmp_path / "rand4.bin"
    f.write_bytes(rng.integers(0, 4, 1 << 16, dtype=np.uint8).tobytes())
    out = tmp_path / "m.csv"
    assert cli.main(["bench", "--text", str(f), "--algos", "B200,HOR,SSEF", "--lengths", "4,32",
                     "--patterns", "3", "--out", str(out)]) == 0
    lines = [ln for ln in out.read_text().splitlines() if not ln.startswith("#")]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    assert tuple(rows[0]) == cli.CSV_HEADER
    cells = {(r[3], int(r[4])) for r in rows[1:]}
    assert cells == {("B200", 4), ("B200", 32), ("HOR", 4), ("HOR", 32), ("SSEF", 32)}  # SSEF m>=32
    assert all(float(r[5]) > 0 and r[8] == "time" and int(r[1]) == 4 for r in rows[1:])


def test_run_benchmark_mirror(cuda):
    import paper_1012_2547_b200 as mb

    text = mb.generate_rand_text(4, 1 << 16, seed=3)
    cfg = mb.BenchConfig(lengths=(4, 32), patterns_per_length=2)
    ms = mb.run_benchmark(cfg, [text], [mb.get_algorithm("B200"), mb.get_algorithm("SSEF")])
    assert {(x.algorithm, x.m) for x in ms} == {("B200", 4), ("B200", 32), ("SSEF", 32)}
    assert all(x.metric == "time" and x.mean_value > 0 and x.runs == 2 and x.sigma == 4 for x in ms)
