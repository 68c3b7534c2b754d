mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "backward or grad or synthetic" 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -5
bash tools/ab_bench.sh base prevb base prevb 2>&1 | tail -4
