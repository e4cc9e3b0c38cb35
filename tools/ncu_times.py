"""Compact per-launch table from an ncu --csv metrics log (tools only).
usage: ncu_times.py LOG.csv [metric ...]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if r[0] == "ID")
want = sys.argv[2:] or ["gpu__time_duration.sum"]
ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
launches = {}
for r in rows:
    if len(r) != len(hdr) or r[0] == "ID":
        continue
    d = launches.setdefault(r[iid], {"name": r[ik]})
    d[r[im]] = r[iv]
for i, d in sorted(launches.items(), key=lambda x: int(x[0])):
    vals = "  ".join(f"{m.split('__')[-1][:18]}={d.get(m, '-')}" for m in want)
    print(f"{i:>4} {d['name'][:48]:48s} {vals}")
