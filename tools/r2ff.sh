mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh fm3 "-DCS_FWD_MINB=3" "blend" > /dev/null 2>&1
bash tools/build_variant.sh fm5 "-DCS_FWD_MINB=5" "blend" > /dev/null 2>&1
bash tools/build_variant.sh bm5 "-DCS_BWD_MINB=5" "blend" > /dev/null 2>&1
bash tools/ab_bench.sh base fm3 fm5 bm5 base fm3 fm5 bm5 2>&1 | tail -8
