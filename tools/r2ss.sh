mkdir -p gpurun_out
CS_LIB_PATH=variants/both.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "discrete or full_size or hull or beyond" 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -5
bash tools/ab_bench.sh base pu1 su1 both base pu1 su1 both 2>&1 | tail -8
