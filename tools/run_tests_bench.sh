timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -s 2>&1 | grep -E "grad rel err|^E  .*(Assert|Error)|passed|failed" > gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt
