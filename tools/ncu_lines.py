"""Top source lines by warp-stall samples from `ncu --page source --print-source cuda,sass --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
path, out, total = None, [], 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            s = int(r[4])
        except ValueError:
            continue
        total += s
        out.append((s, f"{path}:{r[0]}", r[1][:100]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("total stall samples", total)
for s, loc, src in sorted(out, reverse=True)[:n]:
    print(f"{s:7d} {100 * s / max(total, 1):5.1f}%  {loc:18s} {src}")
