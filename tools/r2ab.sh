mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chair.py -q -s -p no:cacheprovider -k "backward or grad or synthetic or chair or beyond" 2>&1 | grep -E "grad rel err|passed|failed" | sed 's/| strict.*//' | tail -12
bash tools/ab_train.sh base aloop base aloop 2>&1 | tail -4
