mkdir -p gpurun_out
bash tools/ab_bench.sh base pb7 pb5 pb8 base pb7 pb5 pb8 2>&1 | tail -8
