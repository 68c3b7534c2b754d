mkdir -p gpurun_out
timeout 900 python tools/mode_diag.py 2>&1 | grep -v worst | tail -8
python tools/cmp_libs.py abvar/prevb.so 2>&1 | tail -9 | head -7
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
