"""Executed-instruction mix per kernel (opcode -> warp instructions) from an ncu report (tools only)."""
import collections
import csv
import io
import subprocess
import sys

rep, kid = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur[1] = r
    elif cur and cur[1]:
        cur[2].append(r)
name, hdr, body = blocks[kid]
i_src, i_ex, i_s = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
mix, stall = collections.Counter(), collections.Counter()
for b in body:
    src = b[i_src].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0].split(".")[0] if src else "?"
    mix[op] += int(b[i_ex] or 0)
    stall[op] += int(b[i_s] or 0)
tot = sum(mix.values())
print(name, "total warp instr", tot)
for op, c in mix.most_common(25):
    print(f"  {op:<10} {c:>12} {c / tot * 100:5.1f}%  stall {stall[op]}")
