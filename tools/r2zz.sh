mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "discrete or full_size or synthetic or near_ties or capacity" 2>&1 | tail -1
python tools/cmp_libs.py abvar/prevs.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base prevs base prevs 2>&1 | tail -4
