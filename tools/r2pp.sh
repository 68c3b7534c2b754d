mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -12
for i in 1 2; do python bench.py --no-cpu-baseline --no-configs --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_bwd_iters_per_s'], d['stage_ms'], d['train_step']['ms_per_step'])"; done
