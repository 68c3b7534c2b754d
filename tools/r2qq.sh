mkdir -p gpurun_out
for v in ps16ds16; do CS_LIB_PATH=variants/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "discrete or full_size or synthetic" 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -5; done
bash tools/ab_bench.sh base ds16 ps16 ps12 ps16ds16 base ds16 ps16 ps12 ps16ds16 2>&1 | tail -10
