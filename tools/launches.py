"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: mean us per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg.setdefault(d["Kernel Name"][:90], []).append(float(d["Metric Value"].replace(",", "")) / 1000)
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v):9.1f} us  {k}")
