"""Top stall lines per kernel from an ncu report's source page (tools only)."""
import csv
import io
import subprocess
import sys

rep, kid = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
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
i_s, i_src, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(int(b[i_s]) for b in body if b[i_s].isdigit())
print(name, "instructions:", len(body), "samples:", tot)
for b in sorted(body, key=lambda b: -int(b[i_s]) if b[i_s].isdigit() else 0)[:top]:
    print(f"{int(b[i_s]) / tot * 100:5.1f}% ex={b[i_ex]:>9} {b[0][-5:]} {b[i_src][:100]}")
