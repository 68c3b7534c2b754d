mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_sharded.py tests/test_gpu_chair.py tests/test_gpu_train_ops.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/bench_lanes.json 2> gpurun_out/bench_lanes.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_lanes.json').read().strip().splitlines()[-1])
print('train', d['train_step']['ms_per_step'], 'chair', d['configs']['config2']['gpu']['ms_per_step'], d['configs']['config2']['gpu']['mean_view_loss_first_last'])"
