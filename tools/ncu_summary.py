"""Key metrics of each kernel in an ncu report (details page)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "DRAM Throughput",
        "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    seen = set()
    print("==", rep.split("/")[-1], rows[1][ki][:70] if len(rows) > 1 else "")
    for r in rows[1:]:
        key = (r[ki], r[mi])
        if r[mi] in WANT and key not in seen:
            seen.add(key)
            print(f"   {r[mi]:36s} {r[vi]:>12s} {r[ui]}")
