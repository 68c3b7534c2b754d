mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh nonp "-DCS_FWD_NONPERSIST" "blend" > /dev/null 2>&1
bash tools/build_variant.sh ps0 "-DCS_FWD_PROD_SLEEP_NS=0" "blend" > /dev/null 2>&1
bash tools/build_variant.sh ps512 "-DCS_FWD_PROD_SLEEP_NS=512" "blend" > /dev/null 2>&1
python tools/cmp_libs.py variants/nonp.so 2>&1 | tail -9 | head -7
CS_LIB_PATH= bash -c 'true'
bash tools/build_variant.sh ws "-DCS_WAIT_STATS" "blend" > /dev/null 2>&1; CS_LIB_PATH=variants/ws.so timeout 300 python tools/wait_stats.py 2>&1 | tail -2
bash tools/ab_bench.sh base nonp ps0 ps512 base > gpurun_out/ab11.txt 2>&1; cat gpurun_out/ab11.txt
