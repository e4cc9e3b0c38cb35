"""GPU: concurrent contexts and the sharded (multi-rank) path on the engine.

* Four host threads, each with its own context and stream, run large
  searches at the same time.  The offsets kernel and the batch pass prologue
  pass a grid barrier; they are cooperative launches, so two contexts cannot
  each hold part of the GPU and spin (the threading contract of the
  reference: compiled searchers are reentrant, pkg/tests/test_registry.py:152-162).
* two ranks (gloo, one process each, both on
  cuda:0 -- their kernels never wait on one another) search their text
  stripes with the CUDA engine and gather the global position list; batched
  mode shards the patterns.
"""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_1012_2547_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_concurrent_contexts_large_searches(cuda):
    n = 2 << 30  # 256 offsets chunks: the co-resident (grid-barrier) offsets mode
    g = torch.Generator(device="cuda").manual_seed(11)
    d = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)
    # denser spots so every search emits positions through both output kernels
    d[1 << 20 : (1 << 20) + 4096] = 7
    d[(1 << 30) : (1 << 30) + 100000] = torch.randint(0, 2, (100000,), dtype=torch.uint8, device="cuda", generator=g)
    h = d.cpu().numpy()
    pats = [bytes([7, 7, 7]), h[5000:5012].tobytes(), h[(1 << 30) + 500 : (1 << 30) + 520].tobytes(),
            h[123456:123456 + 64].tobytes()]
    wants = [oracle.search(p, h, threads=os.cpu_count() or 4) for p in pats]
    # a batch that takes the batch pass (its prologue has the other grid barrier)
    bt = d[: 256 << 20]
    bh = h[: 256 << 20]
    rng = np.random.default_rng(3)
    bpats = [bh[i : i + 24].tobytes() for i in rng.integers(0, bh.size - 24, 300)]
    bwant = [oracle.search(p, bh) for p in bpats[:20]]
    torch.cuda.synchronize()
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            plans = [engine.Plan(p) for p in pats]
            bplans = [engine.Plan(p) for p in bpats]
            mp0 = engine.mp_batches()
            with torch.cuda.stream(s):
                for it in range(3):
                    for j in range(len(pats)):
                        k = (i + j + it) % len(pats)
                        got = engine.find(plans[k], d, stream=s)
                        s.synchronize()
                        if not np.array_equal(got.cpu().numpy(), wants[k]):
                            errors.append((i, it, k))
                    pos, offs = engine.find_batch(bplans, bt, stream=s)
                    s.synchronize()
                    pos = pos.cpu().numpy()
                    for k in range(len(bwant)):
                        if not np.array_equal(pos[offs[k] : offs[k + 1]], bwant[k]):
                            errors.append((i, it, "batch", k))
            if engine.mp_batches() == mp0:
                errors.append((i, "batch pass not taken"))
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append((i, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=500)
        assert not th.is_alive(), "concurrent searches did not finish"
    assert not errors, errors[:10]


def _rank_worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle as orc
    from paper_1012_2547_b200 import engine as eng
    from paper_1012_2547_b200 import shard

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        rng = np.random.default_rng(21)
        n = (40 << 20) + 12345
        text = rng.integers(0, 4, n, dtype=np.uint8)
        pats = [text[i : i + m].tobytes() for i, m in zip(rng.integers(0, n - 2000, 6), (3, 8, 16, 40, 300, 1500))]
        pats.append(b"\x00\x01\x02\x03" * 2)
        res = {}
        for p in pats:
            lo, hi, rhi = shard.shard_bounds(n, len(p), world, rank)
            stripe = torch.from_numpy(text[lo:rhi].copy()).cuda()

            def search(pp, t):
                return eng.find(eng.Plan(pp), t).cpu()

            local, off, total = shard.sharded_search(p, stripe, n, search)
            full = shard.gather_positions(local)
            res[p] = (off, total, bool(np.array_equal(full.numpy(), orc.search(p, text))))
        # batched mode: patterns sharded over the ranks, text replicated
        d = torch.from_numpy(text).cuda()

        def batch(ps, t):
            pos, offs = eng.find_batch([eng.Plan(pp) for pp in ps], t)
            return pos.cpu(), offs

        bpats = [text[i : i + 12].tobytes() for i in rng.integers(0, n - 12, 50)]
        pos, offs = shard.sharded_search_batch(bpats, d, batch)
        pos = pos.numpy()
        bok = all(np.array_equal(pos[offs[k] : offs[k + 1]], orc.search(p, text)) for k, p in enumerate(bpats))
        q.put((rank, res, bok, eng.launch_count()))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), False, 0))


@pytest.mark.timeout(600)
def test_sharded_engine_two_ranks(cuda):
    import multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=500) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    offs = {}
    for rank, res, bok, launches in outs:
        assert isinstance(res, dict), res
        assert bok, f"rank {rank}: batched sharding mismatch"
        assert launches > 0, f"rank {rank} launched no engine kernel"
        for p, (off, total, ok) in res.items():
            assert ok, (rank, len(p))
            offs.setdefault(p, {})[rank] = (off, total)
    for p, by in offs.items():
        assert by[0][0] == 0 and by[0][1] == by[1][1]
