mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh cf1 "-DCS_CULL_FROM=1" "blend" > /dev/null 2>&1
bash tools/build_variant.sh cf2 "-DCS_CULL_FROM=2" "blend" > /dev/null 2>&1
bash tools/build_variant.sh ws1 "-DCS_WAIT_STATS -DCS_CULL_FROM=1" "blend" > /dev/null 2>&1; CS_LIB_PATH=variants/ws1.so timeout 300 python tools/wait_stats.py 2>&1 | tail -2 | head -1
python tools/cmp_libs.py variants/cf1.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base cf1 cf2 base cf1 > gpurun_out/ab17.txt 2>&1; cat gpurun_out/ab17.txt
