"""Stall-reason totals (warp-state samples) over all source lines of an ncu report."""
import csv
import io
import subprocess
import sys

for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, tot = None, {}
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and len(r) > 2 and r[2] == "-":
            for i, name in enumerate(hdr):
                if name.startswith("stall_") and "Not Issued" not in name:
                    try:
                        tot[name] = tot.get(name, 0) + float(r[i] or 0)
                    except ValueError:
                        pass
    s = sum(tot.values()) or 1
    print("==", rep.split("/")[-1])
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
        print(f"   {k:28s} {100 * v / s:5.1f}%")
