mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chair.py -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
python tools/cmp_libs.py abvar/nopair.so 2>&1 | tail -2
bash tools/ab_bench.sh base nopair bp5 bp4 base nopair bp5 bp4 2>&1 | tail -8
