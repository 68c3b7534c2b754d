# A/B of library variants including the config-5 training step: bash tools/ab_train.sh base v1 v2 ...
for v in "$@"; do
  if [ $v = base ]; then unset CS_LIB_PATH; elif [ -f abvar/$v.so ]; then export CS_LIB_PATH=abvar/$v.so; else export CS_LIB_PATH=variants/$v.so; fi
  python bench.py --no-cpu-baseline --no-e2e --no-configs --steps 5 > gpurun_out/abt_$v.log 2>&1
  tail -1 gpurun_out/abt_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['fwd_bwd_iters_per_s'],1), round(d['train_step']['ms_per_step'],2), {k: round(v,4) for k,v in d['stage_ms'].items() if k in ('blend','backward_blend','chain')})"
done
