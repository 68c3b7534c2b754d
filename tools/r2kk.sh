mkdir -p gpurun_out
for i in 1 2; do timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20; done
bash tools/ab_bench.sh base st3 st5 st6 nola base st3 st5 st6 nola 2>&1 | tail -10
