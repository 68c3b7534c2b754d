mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/ab_bench.sh base > gpurun_out/ab4.txt 2>&1; cat gpurun_out/ab4.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -s -k "synthetic or full_size" 2>&1 | grep -E "grad rel err|passed|failed" | cut -c1-200
