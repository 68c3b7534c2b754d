mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh nonp "-DCS_FWD_NONPERSIST" "blend" > /dev/null 2>&1
bash tools/build_variant.sh p5 "-DCS_FWD_STAGES=5" "blend" > /dev/null 2>&1
bash tools/build_variant.sh p3 "-DCS_FWD_STAGES=3" "blend" > /dev/null 2>&1
python tools/cmp_libs.py variants/nonp.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base nonp p5 p3 base > gpurun_out/ab10.txt 2>&1; cat gpurun_out/ab10.txt
