mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s -x > gpurun_out/pytest_gpu_full.log 2>&1
grep -E "grad rel err|passed|failed|Error" gpurun_out/pytest_gpu_full.log | tail -60
tail -3 gpurun_out/smoke.txt
