mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh gsm "-DCS_BWD_G_SMEM" "blend" > /dev/null 2>&1
bash tools/build_variant.sh gsm5 "-DCS_BWD_G_SMEM -DCS_BWD_MINB=5" "blend" > /dev/null 2>&1
bash tools/ab_bench.sh base gsm gsm5 base gsm > gpurun_out/ab15.txt 2>&1; cat gpurun_out/ab15.txt
