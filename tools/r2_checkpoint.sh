# full GPU checkpoint: tests, smoke, default bench, launch list, ncu of the blends
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1200 python bench.py > gpurun_out/bench_ck.json 2> gpurun_out/bench_ck.err
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt
tail -1 gpurun_out/bench_ck.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_bwd_iters_per_s'], d['e2e']['value'], d['stage_ms'], d['roofline']['kernel'], d['roofline']['frac'], d.get('train_step',{}).get('ms_per_step'), d['clocks'])"
bash tools/profile_r02.sh r02k forward2_kernel backward_kernel:1 preprocess_kernel chain_kernel:1 onesweep_kernel:8 duplicate_scan_kernel > /dev/null 2>&1
ls gpurun_out/r02k*
