"""Command line for the GPU engine.

    python -m paper_1012_2547_b200 search --pattern P --text FILE [--algo auto|ID] [--count]
    python -m paper_1012_2547_b200 bench  --text FILE [--algos B200,HOR] [--lengths 2,4,...] [--patterns 400]

`search` mirrors the reference's `matchbench search` (cli.py:139-173): the
same flags, `\\xNN` pattern escapes, `--algo auto` through the selection map
with sigma counted on the device (K0 histogram), one position per line, exit
0 if any occurrence, 1 if none, 2 on error.  The file is read into pinned host
memory and copied to the GPU once.

`bench` runs the reference's time-mode protocol (bench.py:167-238: patterns
sampled per (text, m) with derive_seed(seed, text_id, m), compile untimed, one
warm-up, timed search, mean/pstdev over patterns) on the GPU, timing each
search with CUDA events, and writes the reference's measurement CSV
(report.py CSV_HEADER, 3-significant-digit values) so the rows feed the
reference's own `report` / best-map pipeline unchanged.
"""
from __future__ import annotations

import argparse
import csv
import io
import math
import statistics
import sys
from pathlib import Path

CSV_HEADER = ("text_id", "sigma", "family", "algorithm", "m", "mean", "stddev", "mean_occurrences", "metric")


def parse_pattern_bytes(s: str) -> bytes:
    r"""Literal pattern bytes with \xNN (and standard backslash) escapes (cli.py:91-93 semantics)."""
    return s.encode("latin-1").decode("unicode_escape").encode("latin-1")


def format_value(x: float) -> str:
    """3 significant digits, plain decimal (the reference CSV's number format)."""
    if x == 0:
        return "0"
    if not math.isfinite(x):
        return str(x)
    digits = 2 - math.floor(math.log10(abs(x)))
    y = round(x, digits)
    if digits <= 0:
        return str(int(y))
    s = f"{y:.{digits}f}".rstrip("0").rstrip(".")
    return s if s not in ("", "-") else "0"


def read_text_pinned(path):
    """Raw file bytes -> pinned host tensor -> CUDA tensor (one H2D copy)."""
    import numpy as np
    import torch

    size = Path(path).stat().st_size
    host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    if size:
        with open(path, "rb") as f:
            f.readinto(memoryview(host.numpy()))
    dev = torch.empty(size, dtype=torch.uint8, device="cuda")
    if size:
        dev.copy_(host, non_blocking=True)
    return host, dev


def device_alphabet_size(d_text) -> int:
    from . import engine

    if d_text.numel() == 0:
        return 0
    return int((engine.histogram(d_text) > 0).sum().item())


def cmd_search(args) -> int:
    from .core import ApplicabilityError, Pattern
    from .registry import get_algorithm, select_applicable

    if args.pattern_file:
        raw = Path(args.pattern_file).read_bytes()
    elif args.pattern is not None:
        try:
            raw = parse_pattern_bytes(args.pattern)
        except UnicodeError as exc:
            print(f"error: cannot parse pattern: {exc}", file=sys.stderr)
            return 2
    else:
        print("error: one of --pattern / --pattern-file is required", file=sys.stderr)
        return 2
    try:
        pattern = Pattern(raw)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    _, d_text = read_text_pinned(args.text)
    if args.algo.strip().lower() == "auto":
        algo = select_applicable(max(device_alphabet_size(d_text), 1), len(pattern))
    else:
        try:
            algo = get_algorithm(args.algo)
        except KeyError as exc:
            print(f"error: {exc.args[0]}", file=sys.stderr)
            return 2
    try:
        run = algo.compile(pattern.data)  # bounds enforced here, as in the reference
    except ApplicabilityError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    if len(pattern) > d_text.numel():
        positions = []
    else:
        from . import engine

        pos = engine.find(run.plan, d_text)
        if args.count:
            print(int(pos.numel()))
            return 0 if pos.numel() else 1
        positions = pos.cpu().tolist()
    if args.count:
        print(len(positions))
    else:
        sys.stdout.write("".join(f"{i}\n" for i in positions))
    return 0 if positions else 1


def gpu_benchmark(text_bytes, text_id, algos, lengths, patterns_per_length, seed, warmup=True):
    """Time-mode cells (bench.py:167-238 protocol) measured on the GPU with CUDA events (ms)."""
    import numpy as np
    import torch

    from . import engine
    from .inputs import derive_seed, sample_positions

    t = np.frombuffer(text_bytes, dtype=np.uint8)
    d = torch.from_numpy(t.copy()).cuda()
    sigma = device_alphabet_size(d)
    stream = torch.cuda.current_stream()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    rows = []
    for algo in algos:
        for m in lengths:
            if m > t.size or not algo.applicable(m):
                continue
            pats = [t[i : i + m].tobytes() for i in sample_positions(t.size, m, patterns_per_length,
                                                                      derive_seed(seed, text_id, m))]
            vals, occ = [], 0
            for p in pats:
                run = algo.compile(p)
                plan = run.plan
                out = torch.empty(max(engine.count(plan, d), 1), dtype=torch.int64, device="cuda")
                if warmup:
                    engine.find_into(plan, d, out, cnt, stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                engine.find_into(plan, d, out, cnt, stream)
                e1.record(stream)
                e1.synchronize()
                vals.append(e0.elapsed_time(e1))
                occ += int(cnt.item())
            rows.append((text_id, sigma, algo.family, algo.id, m, statistics.fmean(vals), statistics.pstdev(vals),
                         occ / len(pats), "time"))
    return rows


def sort_rows(rows):
    """Row order of the reference's CSV (report.py:50-51 _row_key): registry
    order, then unknown ids (B200) by name, then m."""
    from .registry import REGISTRY

    order = {a.id: i for i, a in enumerate(REGISTRY)}
    return sorted(rows, key=lambda r: (order.get(r[3], len(order)), r[3], r[4]))


def render_csv(rows) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_HEADER)
    for r in sort_rows(rows):
        w.writerow([r[0], r[1], r[2], r[3], r[4], format_value(r[5]), format_value(r[6]), format_value(r[7]), r[8]])
    return buf.getvalue()


def cmd_bench(args) -> int:
    from .registry import REGISTRY, get_algorithm

    text = Path(args.text).read_bytes()
    text_id = args.id or Path(args.text).stem
    if args.algos.strip().lower() == "all":
        algos = list(REGISTRY)
    else:
        algos = [get_algorithm(a.strip()) for a in args.algos.split(",") if a.strip()]
    lengths = tuple(sorted({int(x) for x in args.lengths.split(",") if x.strip()}))
    rows = gpu_benchmark(text, text_id, algos, lengths, args.patterns, args.seed)
    import numpy as np

    meta = (f"# prng=numpy-pcg64 numpy={np.__version__} seed={args.seed} patterns={args.patterns} metric=time"
            f" text={text_id} n={len(text)} device=cuda engine=b200\n")
    out = meta + render_csv(rows)
    if args.out:
        Path(args.out).write_text(out)
        print(f"wrote {args.out}: {len(rows)} measurements", file=sys.stderr)
    else:
        sys.stdout.write(out)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1012_2547_b200", description="B200 exact string matching engine")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("search", help="print occurrences of a pattern in a file")
    p.add_argument("--algo", default="auto", help="algorithm id (bounds of that id apply), B200, or 'auto'")
    p.add_argument("--pattern", help="pattern; \\xNN escapes accepted")
    p.add_argument("--pattern-file", help="file holding the raw pattern bytes (wins over --pattern)")
    p.add_argument("--text", required=True, help="text file (raw bytes)")
    p.add_argument("--count", action="store_true", help="print the occurrence count only")
    p.set_defaults(func=cmd_search)
    p = sub.add_parser("bench", help="GPU time-mode measurement CSV (reference format)")
    p.add_argument("--text", required=True)
    p.add_argument("--id")
    p.add_argument("--algos", default="B200")
    p.add_argument("--lengths", default="2,4,8,16,32,64,128,256,512,1024")
    p.add_argument("--patterns", type=int, default=400)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--out")
    p.set_defaults(func=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
