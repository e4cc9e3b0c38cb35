"""Static SASS opcode histogram per kernel of libmatchb200.so (cuobjdump -sass).
Shows which kernels carry the TMA bulk copies (UBLKCP), mbarrier traffic
(SYNCS), shared/global vector loads and the integer mix of the filters.
usage: python tools/sass_histogram.py > profiles/r2/sass_histogram.txt"""
import collections
import os
import re
import subprocess
import sys

so = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1012_2547_b200", "libmatchb200.so")
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
dem = {}
kern, hist = None, collections.OrderedDict()
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        hist[kern] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)((?:\.[A-Z0-9_]+)*)", line)
    if m and kern:
        op = m.group(1)
        if op in ("LDS", "LDG", "STG", "STS", "ATOMG", "ATOMS", "RED"):
            w = [x for x in m.group(2).split(".") if x in ("128", "64", "U16", "U8", "16", "8")]
            op += "." + w[0] if w else ""
        hist[kern][op] += 1
names = subprocess.run(["c++filt"], input="\n".join(hist), capture_output=True, text=True).stdout.splitlines()
keys = ["UBLKCP", "SYNCS", "LDS.128", "LDS.64", "LDS", "LDG.128", "LDG", "STG", "STG.64", "ATOMG", "RED", "SHF", "LOP3", "ISETP", "IADD3",
        "IMAD", "PRMT", "POPC", "FLO", "SHFL", "VOTE", "BAR", "MATCH"]
print("kernels:", len(hist))
print("totals:", dict(sum((collections.Counter(h) for h in hist.values()), collections.Counter()).most_common(12)))
print(f"{'kernel':<64} {'instr':>6} " + " ".join(f"{k:>7}" for k in keys))
for (k, h), nm in zip(hist.items(), names):
    short = re.sub(r"\(mb::\w+\)|void |mb::", "", nm)[:64]
    print(f"{short:<64} {sum(h.values()):>6} " + " ".join(f"{h.get(x, 0):>7}" for x in keys))
