"""Per-source-line instructions executed and stall samples from an ncu report.

usage: python tools/ncu_src.py <report.ncu-rep> [N]
Reads `ncu -i R --page source --csv --print-source cuda` (CUDA-source view,
requires -lineinfo) and prints the top lines by warp instructions executed
and by stall samples, with the kernel's totals.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    # source-level rows carry "-" in the Address column; columns by position
    # (the header repeats "Source"): 0 line, 1 source, 2 address, 4 stalls, 7 instructions
    if hdr and len(r) > 7 and r[2] == "-" and r[0] not in ("", "Line No"):
        try:
            ins = float(r[7].replace(",", "") or 0)
            st = float(r[4].replace(",", "") or 0)
        except ValueError:
            continue
        if ins or st:
            rows.append((ins, st, f"{fname}:{r[0]}", r[1].strip()[:90]))
ti = sum(r[0] for r in rows) or 1
ts = sum(r[1] for r in rows) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts:.0f}")
print("-- by instructions")
for ins, st, loc, src in sorted(rows, reverse=True)[:n]:
    print(f"{ins:11.4g} {100 * ins / ti:5.1f}%  st {100 * st / ts:5.1f}%  {loc:16s} {src}")
print("-- by stalls")
for ins, st, loc, src in sorted(rows, key=lambda r: -r[1])[:n]:
    print(f"{ins:11.4g} {100 * ins / ti:5.1f}%  st {100 * st / ts:5.1f}%  {loc:16s} {src}")
