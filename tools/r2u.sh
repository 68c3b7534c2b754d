mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "p4m8:-DCS_BWD_PPL=4 -DCS_BWD_MINB=8" "p4m10:-DCS_BWD_PPL=4 -DCS_BWD_MINB=10" "p4m12:-DCS_BWD_PPL=4 -DCS_BWD_MINB=12" "p2m7:-DCS_BWD_MINB=7"; do
  n=${v%%:*}; f=${v#*:}; bash tools/build_variant.sh $n "$f -Xptxas -v" "blend" > gpurun_out/bv_$n.log 2>&1
  grep -A2 "backward_kernelILi8ELi[24]ELb0" gpurun_out/bv_$n.log | grep -i "spill\|registers" | head -2
done
bash tools/ab_bench.sh base p4m8 p4m10 p4m12 p2m7 > gpurun_out/ab14.txt 2>&1; cat gpurun_out/ab14.txt
