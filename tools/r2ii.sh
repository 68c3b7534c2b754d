mkdir -p gpurun_out
B="bench.py --no-cpu-baseline --no-e2e --no-train --no-configs --steps 1 --warmup 0"
for v in base sl0 sl8k; do
  if [ $v = base ]; then unset CS_LIB_PATH; else export CS_LIB_PATH=abvar/$v.so; fi
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k "regex:forward_kernel|backward_kernel" --csv --log-file gpurun_out/inst_$v.csv python $B > /dev/null 2>&1
  echo $v; python - $v <<'PY'
import csv, sys
lines = [l for l in open(f"gpurun_out/inst_{sys.argv[1]}.csv") if not l.startswith("==")]
rows = list(csv.DictReader(lines))
for r in rows:
    print(r["Kernel Name"][:40], r["Metric Name"], r["Metric Value"])
PY
done
