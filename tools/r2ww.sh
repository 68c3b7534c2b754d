mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chair.py -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -5
python tools/cmp_libs.py abvar/prev2.so 2>&1 | tail -9 | head -7
bash tools/ab_train.sh base prev2 base prev2 2>&1 | tail -4
