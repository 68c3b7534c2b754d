mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
( time timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ) 2> gpurun_out/bench_time.txt
cat gpurun_out/bench_time.txt; tail -5 gpurun_out/bench.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu_full.log
