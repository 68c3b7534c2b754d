mkdir -p gpurun_out
CS_LIB_PATH=variants/dr2sm3.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "discrete or full_size or synthetic or capacity" 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -5
bash tools/ab_bench.sh base dr2 dr1 dr2sm3 dr3 base dr2 dr1 dr2sm3 dr3 2>&1 | tail -10
