"""Summarise an ncu report: per-kernel key metrics + top stall lines (tools only)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Dynamic Shared Memory Per Block", "Grid Size", "Executed Instructions", "L2 Hit Rate", "L1/TEX Hit Rate",
        "No Eligible", "Warp Cycles Per Issued Instruction")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = {k: i for i, k in enumerate(rows[0])}
cur = None
for r in rows[1:]:
    key = (r[h["ID"]], r[h["Kernel Name"]][:60])
    if key != cur:
        cur = key
        print("==", key)
    if r[h["Metric Name"]] in want:
        print(f"   {r[h['Metric Name']]:<38} {r[h['Metric Value']]:>14} {r[h['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr = rr[0]
cols = [i for i, c in enumerate(hdr) if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                                                "Kernel Name", "ID")]
for r in rr[2:]:
    print("raw", [(hdr[i], r[i]) for i in cols])
