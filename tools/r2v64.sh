mkdir -p gpurun_out
python tools/cmp_libs.py abvar/prevb.so 2>&1 | tail -9 | head -7
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "beyond_six or scaling_modes" 2>&1 | grep -E "grad rel err|passed|failed" | sed "s/| strict.*//" | cut -c1-220
timeout 600 python tools/mode_timing.py 2>&1 | tail -4
