#!/usr/bin/env python
"""Headline benchmark: text GB/s scanned (all matches emitted) and % of the HBM roofline.

Workload (default, BASELINE.json config 4 -- the config the north-star roofline
target is quoted on): a 16 GiB i.i.d. uniform sigma=256 text resident in HBM,
one pattern per m in {2, 8, 32, 128, 1024} copied from a random text offset.
A step scans the whole text once per pattern through the C ABI (mb_find) and
writes every position to HBM.  Other configs are parity cases (tests/), or
`--workload cfg1|cfg2|cfg3|cfg5` for ad-hoc runs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: each rank scans its own 16 GiB
stripe of one (N x 16 GiB) text (weak scaling; a (m-1)-byte halo keeps
boundary matches exact) and the ranks all_gather their counts (NCCL) to place
their positions in the global output -- the path's only exchange.
`--impl reference` times the reference algorithms' CPU restatement (oracle/,
the auto-selected searcher per m, all host threads) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPIN_CYCLES = 400_000  # ~0.2 ms at 1.965 GHz: covers the host enqueue of one search / batch

METRIC = "text GB/s scanned (all matches emitted) vs m and σ; % of HBM roofline"
CFG4_LENGTHS = (2, 8, 32, 128, 1024)
PEAK_FALLBACK = 6650.0  # B200_PROFILING.md fallback, GB/s
BACKEND = os.environ.get("MB_BENCH_BACKEND", "nccl")  # gloo only for multi-rank tests on one GPU


FLUSH_DESC = ("L2 flushed before every timed launch: 256 MiB write (evicts the text), then a 256 MiB read of a "
              "second buffer (evicts the write's dirty lines, so their write-back is not charged to the search)")


class L2Flush:
    """Evict the 126 MB L2 between timed launches of L2-sized inputs.  A write
    alone leaves L2 full of dirty lines whose write-back then lands inside the
    next timed launch (measured: +14 us on a 256 MiB scan, tools/flush_modes.py);
    reading a clean buffer afterwards leaves only clean lines."""

    def __init__(self, dev):
        import torch

        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(32 << 20, dtype=torch.int64, device=dev)
        self.sink = torch.empty((), dtype=torch.int64, device=dev)

    def __call__(self):
        import torch

        self.w.zero_()
        torch.sum(self.r, dim=0, out=self.sink)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("cfg4", "cfg1", "cfg2", "cfg3", "cfg3b", "cfg5"), default="cfg4")
    ap.add_argument("--text-bytes", dest="n", type=int, default=0, help="text bytes per GPU (default: the config's size)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--family", default="auto", help="force a kernel family where it applies (experiments)")
    return ap.parse_args()


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (copy)"
    except Exception:
        return PEAK_FALLBACK, "B200_PROFILING.md fallback"


def ncu_traffic(workload, alg_bytes_per_launch):
    """DRAM bytes per launch of the dominant kernel: the ncu-measured ratio of
    traffic to algorithmic bytes (profiles/ncu_summary.json) at this launch size."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f).get(workload, {})
        ratio = d["dram_bytes_per_launch"] / d["algorithmic_bytes_per_launch_min"]
        return int(round(ratio * alg_bytes_per_launch))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workloads
def cfg4_desc(n):
    return (f"cfg4: {n / 2**30:.0f} GiB i.i.d. uniform sigma=256 text per GPU, 1 pattern per m in "
            f"{list(CFG4_LENGTHS)} copied from a random offset")


def _pin(a):
    """numpy -> host tensor, page-locked when a GPU driver is present (the
    reference arm runs on hosts without one)."""
    import torch

    t = torch.from_numpy(a)
    return t.pin_memory() if torch.cuda.is_available() else t


def build_workload(args, rank, world):
    """Host text (pinned) + patterns for this rank; returns dict."""
    import numpy as np
    import torch

    from paper_1012_2547_b200 import inputs

    if args.workload == "cfg4":
        n = args.n or (16 << 30)
        n = (n // inputs.STRIPE) * inputs.STRIPE if n >= inputs.STRIPE else n
        halo = 1023 if rank < world - 1 else 0
        try:
            host = torch.empty(n + halo, dtype=torch.uint8, pin_memory=torch.cuda.is_available())
        except RuntimeError:  # pinned host memory exhausted (many ranks on one node): pageable
            host = torch.empty(n + halo, dtype=torch.uint8)
        h = host.numpy()
        stripe0 = rank * max(n // inputs.STRIPE, 1)
        _cfg4_stripes(h[:n], stripe0, n)
        if halo:
            nxt = np.empty(inputs.STRIPE if n >= inputs.STRIPE else n, dtype=np.uint8)
            _cfg4_stripes(nxt, stripe0 + max(n // inputs.STRIPE, 1), nxt.size)
            h[n:] = nxt[:halo]
        pats = inputs.config4_patterns(h[:n]) if rank == 0 else None
        desc = cfg4_desc(n)
        sigma = 256
    elif args.workload == "cfg1":
        t, pats = inputs.config1()
        n, halo = t.size, 0
        host = _pin(t)
        desc = "cfg1: 1 MiB sigma=4, one m=8 pattern"
        sigma = 4
    elif args.workload == "cfg3":
        n = args.n or (64 << 20)
        t = inputs.zipf_text(n, inputs.derive_seed(inputs.ROOT_SEED, "cfg3", "text"))
        host, halo = _pin(t), 0
        pats = [inputs.config3_patterns(t, m, 1)[0] for m in (4, 16, 64, 256, 1024)]
        desc = "cfg3: 64 MiB Zipf text (95 printable symbols), 1 pattern per m in [4,16,64,256,1024]"
        sigma = 95
    else:  # cfg5
        n = args.n or (256 << 20)
        t = inputs.dense_text(n, inputs.derive_seed(inputs.ROOT_SEED, "cfg5", "text"))
        host, halo = _pin(t), 0
        pats = inputs.config5_patterns()
        desc = "cfg5: 256 MiB 99.9% 'a' text, patterns a^m and a^(m-1)b for m in [2,16,128,1024]"
        sigma = 26
    if world > 1:
        import torch.distributed as dist

        obj = [pats]
        dist.broadcast_object_list(obj, src=0)
        pats = obj[0]
    return {"host": host, "n": n, "halo": halo, "patterns": pats, "desc": desc, "sigma": sigma}


def _cfg4_stripes(out, first_stripe, n):
    import concurrent.futures as cf

    from paper_1012_2547_b200 import inputs

    S = inputs.STRIPE
    k = max((n + S - 1) // S, 1)

    def one(i):
        lo, hi = i * S, min(n, (i + 1) * S)
        inputs.rand_text_np(256, hi - lo, inputs.derive_seed(inputs.ROOT_SEED, "cfg4", "text", first_stripe + i),
                            out=out[lo:hi])

    with cf.ThreadPoolExecutor(min(32, os.cpu_count() or 4)) as ex:
        list(ex.map(one, range(k)))


# ------------------------------------------------------------------ reference arm
def run_config(args, wl, world, flush):
    """The `config` object both arms print (identical for identical workloads)."""
    return {"workload": wl["desc"], "text_bytes_per_gpu": int(wl["n"]), "patterns_m": [len(p) for p in wl["patterns"]],
            "l2": "inputs larger than L2 (text > 4x 126 MB), no flush needed" if not flush
            else FLUSH_DESC + "; ms = sum of launch events",
            "parallelism": f"dp{world} (text stripes, count all_gather)"}


def run_reference(args, rank, world):
    """The reference's algorithms (CPU restatement in oracle/, auto-selected per
    m as `matchbench search --algo auto` does, registry.py:209-222) on all host
    threads, over the SAME workload as our arm: the same text (the whole
    16 GiB for config 4), the same patterns, every position emitted into host
    memory (the oracle's threaded driver scans each chunk once and grows its
    output buffers).  Rank 0 only; the other ranks exit without work."""
    if rank != 0:
        return
    import oracle
    from paper_1012_2547_b200.registry import select_applicable

    threads = os.cpu_count() or 1
    wl = build_workload(args, 0, 1)
    n = wl["n"]
    t = wl["host"].numpy()[:n]
    pats, sigma = wl["patterns"], wl["sigma"]
    algos = [select_applicable(sigma, len(p)).id for p in pats]

    def step():
        tot = 0
        for p, a in zip(pats, algos):
            tot += oracle.search(p, t, a, threads=threads).size
        return tot

    # one warm-up pass is all a CPU scan needs (page-in, thread start); more
    # would only stretch the run past a few minutes at 16 GiB per pattern
    warm = min(args.warmup, 1)
    for _ in range(warm):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        found = step()
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    value = len(pats) * n / dt / 1e9  # the host's throughput (rank 0's stripe; more stripes take proportionally longer)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": warm, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": run_config(args, wl, world, wl["n"] + wl["halo"] <= (512 << 20)),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"the whole workload: {n / 2**30:.2f} GiB x {len(pats)} patterns per step, "
                                   f"every position emitted ({found} per step), algorithms {algos} "
                                   f"(oracle/oracle.c restatement of the reference's auto path, {threads} threads "
                                   f"over halo-overlapped chunks)"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(wl, sample_bytes):
    """Single-core reference-path baseline on a bounded prefix (bench.py:171-181
    time-mode semantics: compile untimed, 1 warm-up, timed run)."""
    import oracle
    from paper_1012_2547_b200.registry import select_applicable

    t = wl["host"].numpy()[: min(wl["n"], sample_bytes)]
    total_t, total_b, used = 0.0, 0, []
    for p in wl["patterns"]:
        a = select_applicable(wl["sigma"], len(p)).id
        oracle.count(p, t[: 1 << 20], a)  # warm-up
        t0 = time.perf_counter()
        oracle.count(p, t, a)
        total_t += time.perf_counter() - t0
        total_b += t.size
        used.append(a)
    return {"value": round(total_b / total_t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{t.size / 2**20:.0f} MiB prefix x {len(wl['patterns'])} patterns, reference auto path "
                      f"{used} restated in C (oracle/), 1 thread of {os.cpu_count()} host cores"}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_1012_2547_b200 import engine

    dist = None
    if world > 1:
        import torch.distributed as dist
    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    wl = build_workload(args, rank, world)
    n, halo, pats = wl["n"], wl["halo"], wl["patterns"]
    d_text = torch.empty(n + halo, dtype=torch.uint8, device=dev)
    d_text.copy_(wl["host"], non_blocking=False)
    plans = [engine.Plan(p) for p in pats]
    views = [d_text[: min(n + len(p) - 1, n + halo)] for p in pats]  # starts < n on this rank
    # output capacity: count first (untimed), then allocate
    cnts = [engine.count(pl, v) for pl, v in zip(plans, views)]
    out = torch.empty(max(max(cnts), 1), dtype=torch.int64, device=dev)
    cnt = torch.zeros(len(plans), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    K = len(plans)
    # texts up to 4x the 126 MB L2 are flushed out of L2 (L2Flush, outside
    # the per-launch events) before every timed launch; ms_per_step is then the
    # sum of the launches' event durations
    flush = L2Flush(dev) if n + halo <= (512 << 20) else None

    def step(ev=None):
        for i, (pl, v) in enumerate(zip(plans, views)):
            if ev is not None and flush is not None:
                flush()
                torch.cuda._sleep(SPIN_CYCLES)  # GPU busy while the host enqueues the search
            if ev is not None:
                ev[i][0].record(stream)
            engine.find_into(pl, v, out, cnt[i : i + 1], stream)
            if ev is not None:
                ev[i][1].record(stream)
        if dist is not None:  # exchange: global output offsets from per-rank counts
            src = cnt if BACKEND == "nccl" else cnt.cpu()
            allc = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(allc, src)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(K)]
           for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clk:
        clk.start()
        time.sleep(0.25)
    l0 = engine.launch_count()
    torch.cuda.synchronize()
    t_start.record(stream)
    for s in range(args.steps):
        step(evs[s])
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches = engine.launch_count() - l0
    clocks = clk.stop() if clk else None
    ms = t_start.elapsed_time(t_end) / args.steps
    if flush is not None:
        ms = sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(args.steps) for i in range(K)) / args.steps
    if dist is not None:
        tt = torch.tensor([ms], device=dev if BACKEND == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    counts = cnt.cpu().tolist()
    per_launch = [[evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(args.steps)] for i in range(K)]
    bytes_scanned = [v.numel() for v in views]
    value = world * sum(min(b, n) for b in bytes_scanned) / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel (the full-scan scan_kernel, HBM-bound):
    # algorithmic bytes n + 8*count + 8 per launch / its CUDA-event duration.
    # Sampled-q-gram launches (K3) read one 128-byte DRAM line per S text bytes;
    # they are reported per m with that traffic model instead.
    infos = [pl.info() for pl in plans]
    peak, peak_src = measured_peak()
    avg_ms = [statistics.mean(x) for x in per_launch]
    full = [i for i, inf in enumerate(infos) if inf.family != "sampled"]
    per_m = []
    for i, (p, c, a, b) in enumerate(zip(pats, counts, avg_ms, bytes_scanned)):
        inf = infos[i]
        if inf.family == "sampled":
            alg = -(-b // inf.stride) * 128 + 8 * c + 8
        else:
            alg = b + 8 * c + 8
        per_m.append({"m": len(p), "family": inf.family, "count": c, "ms": round(a, 4),
                      "text_gbps": round(b / (a * 1e-3) / 1e9, 1),
                      "alg_bytes": int(alg), "hbm_frac": round((alg / (a * 1e-3) / 1e9) / peak, 4),
                      **({"stride": inf.stride, "gram": inf.gram} if inf.family == "sampled" else {})})
    sel = full if full else list(range(K))
    achieved = sum(per_m[i]["alg_bytes"] for i in sel) / (sum(avg_ms[i] for i in sel) * 1e-3) / 1e9
    traffic = ncu_traffic(args.workload, statistics.mean(per_m[i]["alg_bytes"] for i in sel))

    parity = None
    if not args.no_parity and rank == 0:
        import oracle

        h = wl["host"].numpy()
        ok = True
        for i, (p, v) in enumerate(zip(pats, views)):
            want = oracle.search(p, h[: v.numel()], "BF", threads=os.cpu_count() or 1)
            engine.find_into(plans[i], v, out, cnt[i : i + 1], stream)
            got = out[: int(cnt[i].item())].cpu().numpy()
            ok = ok and np.array_equal(got, want)
        parity = "bit-exact vs oracle (all positions, all patterns)" if ok else "MISMATCH"

    e2e = None
    if not args.no_e2e:
        # reference-facing C ABI with HOST buffers: H2D of the text, scan of all
        # patterns, D2H of every position -- inside the timed region
        host_np = wl["host"].numpy()[:n]  # single-GPU host entry has no halo semantics
        total_pos = sum(cnts) if world == 1 else sum(cnts)
        h_out = torch.empty(max(total_pos, 1), dtype=torch.int64, pin_memory=True).numpy()
        h_offs = np.zeros(K + 1, dtype=np.int64)
        engine.search_batch_host(pats, host_np, h_out, h_offs)  # warm-up (buffers, plans)
        times = []
        for _ in range(max(args.e2e_steps, 1)):
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            rc = engine.search_batch_host(pats, host_np, h_out, h_offs)
            times.append(time.perf_counter() - t0)
        dt = statistics.median(times)
        if dist is not None:
            tt = torch.tensor([dt], device=dev if BACKEND == "nccl" else "cpu", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e = {"value": round(world * K * n / dt / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(n + sum(map(len, pats))),
               "d2h_bytes_per_step": int(8 * int(h_offs[-1]) + 8 * (K + 1)), "ms_per_step": round(dt * 1e3, 2),
               "api": "mb_search_batch_host (C ABI, pinned host text in, host positions out)", "rc": int(rc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, 1 << 30)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": run_config(args, wl, world, flush is not None),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                         "traffic_source": "not measured in this run: the ncu-measured DRAM/algorithmic byte ratio "
                                           "of this kernel (profiles/ncu_summary.json) x this run's algorithmic bytes",
                         "kernel": "scan_kernel (full-scan families, per-pattern launch incl. offsets+expand)",
                         "launches_in_roofline": [len(pats[i]) for i in sel],
                         "algorithmic_bytes": "n + 8*count + 8 per launch (SURVEY.md 8(d))"},
            "per_m": per_m,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)


def run_batched_sweep(args, rank, world, local_rank):
    """Configs 2 and 3 in batched mode: one launch scans the text for all 500
    patterns of a cell (CSR output).  cfg2: 7 sigma x 10 m cells over 4 MiB
    texts; cfg3b: 5 m over the 64 MiB Zipf text.  Value = sum(K * n) / time."""
    import numpy as np
    import torch

    from paper_1012_2547_b200 import engine, inputs

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    cells = []
    if args.workload == "cfg2":
        for sigma in (2, 4, 8, 16, 32, 64, 128):
            t = inputs.config2_text(sigma)
            for m in inputs.DEFAULT_LENGTHS:
                cells.append((sigma, m, t, inputs.config2_patterns(t, sigma, m)))
    else:
        t = inputs.config3()
        for m in (4, 16, 64, 256, 1024):
            cells.append((95, m, t, inputs.config3_patterns(t, m)))
    flush = L2Flush(dev)
    rows, tot_b, tot_alg, tot_ms, launches0 = [], 0, 0, 0.0, engine.launch_count()
    peak, peak_src = measured_peak()
    dtexts = {}
    for sigma, m, t, pats in cells:
        key = id(t)
        if key not in dtexts:
            dtexts[key] = torch.from_numpy(t).to(dev)
        d = dtexts[key]
        plans = []
        for p in pats:
            try:
                plans.append(engine.Plan(p, args.family))
            except ValueError:
                plans.append(engine.Plan(p))
        plans = engine.Batch(plans)  # compile once (plans, tables) -- untimed, as the reference's compile step
        offs = torch.zeros(len(plans) + 1, dtype=torch.int64, device=dev)
        engine.find_batch_into(plans, d, None, offs, stream)  # count pass sizes the output (untimed)
        total = int(offs[-1].item())
        out = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
        for _ in range(max(args.warmup, 3)):
            engine.find_batch_into(plans, d, out, offs, stream)
        # L2 flushed before every timed launch (the text is L2-sized): each rep
        # starts with the text in HBM, as a one-off search would
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for e0, e1 in evs:
            flush()
            torch.cuda._sleep(SPIN_CYCLES)  # GPU busy while the host enqueues the batch: device time only
            e0.record(stream)
            engine.find_batch_into(plans, d, out, offs, stream)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
        b = len(pats) * t.size
        fams = sorted({pl.info().family for pl in plans.plans})
        # batched-mode algorithmic bytes: the text once for the whole
        # batch, every pattern, 8 B per position, the K + 1 CSR offsets
        alg = t.size + sum(len(p) for p in pats) + 8 * total + 8 * (len(pats) + 1)
        rows.append({"sigma": sigma, "m": m, "patterns": len(pats), "ms": round(ms, 4),
                     "text_gbps": round(b / (ms * 1e-3) / 1e9, 1), "matches": total, "families": fams,
                     "alg_bytes": alg, "hbm_frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4)})
        tot_b += b
        tot_alg += alg
        tot_ms += ms
    value = tot_b / (tot_ms * 1e-3) / 1e9
    achieved = tot_alg / (tot_ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(tot_ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{args.workload}: batched, 500 patterns per launch (CSR)",
                       "l2": FLUSH_DESC + "; value aggregated K*n/t",
                       "timing": "per cell: median of the steps' CUDA-event times; a spin kernel keeps the "
                                 "GPU busy while each launch is enqueued, so host enqueue time is excluded"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                         "kernel": "whole batched launches (batch pass / per-pattern scans, offsets, expand, replicate)",
                         "algorithmic_bytes": "n + sum(m_k) + 8 * sum(count_k) + 8 * (K + 1) per batch (SURVEY.md 8(d)): "
                                              "the text read once for the whole batch"},
            "cells": rows, "gpu_launches": engine.launch_count() - launches0}), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank % torch.cuda.device_count())
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # MB_BENCH_BACKEND=gloo: multi-rank plumbing test with ranks sharing GPUs
            dist.init_process_group("gloo")
    try:
        if args.workload in ("cfg2", "cfg3b"):
            run_batched_sweep(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
