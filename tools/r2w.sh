mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh nola "-DCS_NO_LOOK_AHEAD" "blend" > /dev/null 2>&1
bash tools/build_variant.sh ws "-DCS_WAIT_STATS" "blend" > /dev/null 2>&1; CS_LIB_PATH=variants/ws.so timeout 300 python tools/wait_stats.py 2>&1 | tail -2
python tools/cmp_libs.py variants/nola.so 2>&1 | tail -9 | head -8
bash tools/ab_bench.sh base nola base nola > gpurun_out/ab16.txt 2>&1; cat gpurun_out/ab16.txt
