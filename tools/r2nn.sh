mkdir -p gpurun_out
python tools/cmp_libs.py abvar/p4m7.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base p4m7 p4m6 p4m5 base p4m7 p4m6 p4m5 2>&1 | tail -8
