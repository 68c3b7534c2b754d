mkdir -p gpurun_out
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -12; done
