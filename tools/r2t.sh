mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
bash tools/ab_bench.sh head base head base > gpurun_out/ab13.txt 2>&1; cat gpurun_out/ab13.txt
