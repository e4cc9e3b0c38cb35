"""How the L2 flush before a timed launch affects mid-size texts (tools only).

A write flush (zero_ of a buffer > L2) leaves L2 full of DIRTY lines that the
timed scan then writes back to HBM; a read of a second clean buffer after it
leaves only clean lines.  Prints per-search device time for each mode."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1012_2547_b200 import engine, inputs  # noqa: E402

SPIN = 400_000
dev = torch.device("cuda", 0)
wflush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rflush = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
sink = torch.empty(1, dtype=torch.int64, device=dev)


def mode_flush(mode):
    if mode in ("write", "write+read"):
        wflush.zero_()
    if mode in ("read", "write+read"):
        torch.sum(rflush.view(torch.int64), dim=0, out=sink)


for n, pat_m in ((1 << 20, 8), (64 << 20, 16), (256 << 20, 16), (1 << 30, 16)):
    t = inputs.rand_text_np(256, n, 7)
    d = torch.from_numpy(t).to(dev)
    pl = engine.Plan(t[12345:12345 + pat_m].tobytes())
    out = torch.empty(1 << 16, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(5):
        engine.find_into(pl, d, out, cnt)
    for mode in ("none", "write", "read", "write+read"):
        ts = []
        for _ in range(15):
            mode_flush(mode)
            torch.cuda._sleep(SPIN)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            engine.find_into(pl, d, out, cnt)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        med = statistics.median(ts)
        print(f"n={n >> 20:5d} MiB m={pat_m:3d} flush={mode:10s} median {med:8.1f} us  min {min(ts):8.1f} us  "
              f"{n / (med * 1e-6) / 1e9:8.1f} GB/s", flush=True)
