mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
python tools/cmp_libs.py abvar/head.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base head base head 2>&1 | tail -4
bash tools/ab_train.sh base head 2>&1 | tail -2
