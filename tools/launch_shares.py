"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv); tools only."""
import collections
import csv
import sys

rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows))
h = r[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for row in r[1:]:
    try:
        per[(row[iid], row[ik])][row[im]] = float(row[iv].replace(",", ""))
    except ValueError:
        pass
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, k), d in per.items():
    name = k.split("(")[0].replace("void ", "")[:48]
    a = agg[name]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0)
    a[3] += d.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values()) or 1
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    unit = 1e-3  # ns -> us
    print(f"{name:<50} n={a[0]:>3} share={100 * a[1] / tot:5.1f}% avg={a[1] / a[0] * unit:9.1f}us "
          f"rd/launch={a[2] / a[0]:.3e} wr/launch={a[3] / a[0]:.3e}")
