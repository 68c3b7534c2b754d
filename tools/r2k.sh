mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "s0:-DCS_PROD_SLEEP_NS=0" "s256:-DCS_PROD_SLEEP_NS=256" "s2048:-DCS_PROD_SLEEP_NS=2048"; do
  n=${v%%:*}; f=${v#*:}; bash tools/build_variant.sh $n "$f" "blend" > /dev/null 2>&1
done
bash tools/ab_bench.sh head base s0 s256 s2048 head base > gpurun_out/ab6.txt 2>&1; cat gpurun_out/ab6.txt
