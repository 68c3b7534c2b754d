# per-launch device times of one forward+backward frame (ncu, serialized): bash tools/launch_list.sh <tag>
tag=${1:-ll}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-train > gpurun_out/${tag}_launches.log 2>&1
python - "$tag" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/{sys.argv[1]}_launches.csv")))
hdr, seq = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            seq.append((d["Kernel Name"][:50], float(d["Metric Value"].replace(",", "")) / 1000))
for k, v in seq[:24]:
    print(f"{v:8.1f} {k}")
PY
