mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "s0:-DCS_PROD_SLEEP_NS=0" "s256:-DCS_PROD_SLEEP_NS=256" "s1024:-DCS_PROD_SLEEP_NS=1024" "s2048:-DCS_PROD_SLEEP_NS=2048"; do
  n=${v%%:*}; f=${v#*:}; bash tools/build_variant.sh $n "$f" "blend" > /dev/null 2>&1
done
sed -i 's/--no-e2e --steps 10/--no-e2e --no-configs --steps 10/' tools/ab_bench.sh
bash tools/ab_bench.sh base s0 s256 s1024 s2048 > gpurun_out/ab5.txt 2>&1; cat gpurun_out/ab5.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x 2>&1 | tail -2
