for v in base vsort vpre vblend; do
  if [ $v = base ]; then unset CS_LIB_PATH; else export CS_LIB_PATH=abvar/$v.so; fi
  python bench.py --no-cpu-baseline --no-configs --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['fwd_bwd_iters_per_s'], d['train_step']['ms_per_step'])"
done
