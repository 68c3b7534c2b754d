# A/B the stage times of library variants: bash tools/ab_bench.sh base v1 v2 ...
for v in "$@"; do
  if [ $v = base ]; then unset CS_LIB_PATH; elif [ -f abvar/$v.so ]; then export CS_LIB_PATH=abvar/$v.so; else export CS_LIB_PATH=variants/$v.so; fi
  python bench.py --no-cpu-baseline --no-train --no-e2e --no-configs --steps 10 > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['fwd_bwd_iters_per_s'],1), {k: round(v,4) for k,v in d['stage_ms'].items()})"
done
