"""Per-CUDA-source-line instruction and stall totals from an ncu report (tools only).
usage: ncu_lines_cuda.py REPORT [KERNEL_INDEX] [TOP] [NORM]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
norm = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines = "", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        lines.append((fname, r))
iex, iss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot_ex = sum(int(r[iex]) for _, r in lines if r[iex].isdigit())
tot_ss = sum(int(r[iss]) for _, r in lines if r[iss].isdigit())
print(f"total warp instructions {tot_ex} ({tot_ex / norm:.1f} per unit), samples {tot_ss}")
for f, r in sorted(lines, key=lambda x: -int(x[1][iss]) if x[1][iss].isdigit() else 0)[:top]:
    print(f"{int(r[iss]) / max(tot_ss, 1) * 100:5.1f}% ex/unit={int(r[iex]) / norm:7.1f} {f}:{r[0]:<4} {r[1].strip()[:90]}")
