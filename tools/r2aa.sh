mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; tail -1 gpurun_out/pytest_gpu_full.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['fwd_bwd_iters_per_s'], d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['train_step']['ms_per_step'], d['configs']['config2']['gpu']['ms_per_step'], d['clocks'])"
