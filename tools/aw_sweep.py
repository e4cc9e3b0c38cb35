"""Config-2 cells timed with the ALIGNED anchor forced to 1/2/3 words and on
auto (tuning MB_ALIGNED2_RATE / MB_ALIGNED3_RATE); counts cross-checked."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_1012_2547_b200 import engine, inputs

def timed(obj, d, out, offs, reps=5):
    for _ in range(2): engine.find_batch_into(obj, d, out, offs)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    torch.cuda.synchronize(); ev[0].record()
    for i in range(reps):
        engine.find_batch_into(obj, d, out, offs)
        ev[i + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    return ts[reps // 2] if ts[-1] < 1.5 * ts[0] else (ts[reps // 2], ts)

rows = []
for sigma in map(int, (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,16").split(",")):
    t = inputs.config2_text(sigma); d = torch.from_numpy(t).cuda()
    for m in (8, 16, 32, 64, 128, 256):
        pats = inputs.config2_patterns(t, sigma, m)
        ref = None; cell = {"sigma": sigma, "m": m}
        for nw in (0, 1, 2, 3):
            if 4 * nw + 3 > m: continue
            plans = [engine.Plan(p, anchor_words=nw) for p in pats]
            b = engine.Batch(plans)
            offs = torch.zeros(len(plans) + 1, dtype=torch.int64, device="cuda")
            engine.find_batch_into(b, d, None, offs); tot = int(offs[-1])
            out = torch.empty(max(tot, 1), dtype=torch.int64, device="cuda")
            ms = timed(b, d, out, offs)
            c = offs.cpu()
            if ref is None: ref = c
            assert torch.equal(c, ref), (sigma, m, nw)
            key = "auto" if nw == 0 else f"nw{nw}"
            cell[key] = round(ms, 4) if isinstance(ms, float) else [round(ms[0], 4), [round(x, 3) for x in ms[1]]]
            if nw == 0: cell["auto_words"] = sorted({p.info().words for p in plans})
        rows.append(cell); print(json.dumps(cell), flush=True)
json.dump(rows, open("gpurun_out/aw_sweep.json", "w"))
