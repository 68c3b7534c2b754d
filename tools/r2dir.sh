mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "beyond_six or scaling_modes or full_size or synthetic" 2>&1 | grep -E "grad rel err|passed|failed" | sed "s/| strict.*//" | cut -c1-200
bash tools/ab_bench.sh base dir32 base dir32 2>&1 | tail -4
