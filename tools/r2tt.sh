mkdir -p gpurun_out
CS_LIB_PATH=variants/fnl4.so python tools/cmp_libs.py build/../paper_2411_14974_b200/libconvexsplat_sm100.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base fnl4 base fnl4 2>&1 | tail -4
