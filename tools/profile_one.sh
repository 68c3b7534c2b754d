# usage: bash tools/profile_one.sh <kernel-regex> <tag>
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -c 1 -o "gpurun_out/prof_$2" \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "gpurun_out/prof_$2.log" 2>&1
