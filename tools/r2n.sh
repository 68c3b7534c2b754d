mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "sred:-DCS_BWD_SMEM_REDUCE" "sred5:-DCS_BWD_SMEM_REDUCE -DCS_BWD_MINB=5" "sred5s5:-DCS_BWD_SMEM_REDUCE -DCS_BWD_MINB=5 -DCS_BWD_STAGES=5" "sred4:-DCS_BWD_SMEM_REDUCE -DCS_BWD_MINB=4"; do
  n=${v%%:*}; f=${v#*:}; bash tools/build_variant.sh $n "$f" "blend" > gpurun_out/bv_$n.log 2>&1
done
bash tools/ab_bench.sh base sred sred5 sred5s5 sred4 base > gpurun_out/ab8.txt 2>&1; cat gpurun_out/ab8.txt
