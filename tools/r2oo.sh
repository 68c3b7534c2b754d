mkdir -p gpurun_out
for i in 1 2 3 4; do timeout 600 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "synthetic_scene and 131k" 2>&1 | grep -E "grad rel err|passed|failed" | sed 's/| strict.*//'; done
bash tools/ab_bench.sh base f32acc base f32acc 2>&1 | tail -4
