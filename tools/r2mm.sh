mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chair.py -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
bash tools/ab_bench.sh base bs4 bs3 bs5m5 base bs4 bs3 bs5m5 2>&1 | tail -8
