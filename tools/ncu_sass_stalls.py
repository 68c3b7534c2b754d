"""Top SASS instructions per stall reason: python tools/ncu_sass_stalls.py <rep> [reason ...]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reasons = sys.argv[2:] or ["long_sb", "wait", "short_sb", "barrier"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr, rows = None, []
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rows.append(r)
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
src = hdr.index("Source")
for name in reasons:
    ii = hdr.index("stall_" + name)
    top = sorted(rows, key=lambda r: -num(r[ii]))[:8]
    print("==", name)
    for r in top:
        print(f"  {num(r[ii]):7.0f}  {r[0]}  {r[src][:90]}")
