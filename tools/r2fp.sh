mkdir -p gpurun_out
python tools/cmp_libs.py abvar/prevb.so 2>&1 | tail -9 | head -7
CS_LIB_PATH=variants/fnp0.so python tools/cmp_libs.py abvar/prevb.so 2>&1 | tail -9 | head -3
bash tools/ab_train.sh base prevb fnp0 base prevb fnp0 2>&1 | tail -6
