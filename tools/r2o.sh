mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh nonp "-DCS_FWD_NONPERSIST" "blend" > /dev/null 2>&1
timeout 300 python tools/fwd_small.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/ab_bench.sh base nonp base nonp > gpurun_out/ab9.txt 2>&1; cat gpurun_out/ab9.txt
