mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "b5:-DCS_BWD_MINB=5" "b4:-DCS_BWD_MINB=4" "b5s8:-DCS_BWD_MINB=5 -DCS_BWD_STAGES=8" "b5s4:-DCS_BWD_MINB=5 -DCS_BWD_STAGES=4"; do
  n=${v%%:*}; f=${v#*:}; bash tools/build_variant.sh $n "$f" "blend" > gpurun_out/bv_$n.log 2>&1
  grep -A2 "backward_kernelILi8ELi2ELb0" gpurun_out/bv_$n.log | head -3
done
bash tools/ab_bench.sh base b5 b4 b5s8 b5s4 base > gpurun_out/ab7.txt 2>&1; cat gpurun_out/ab7.txt
