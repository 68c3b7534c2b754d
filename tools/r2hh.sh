mkdir -p gpurun_out
bash tools/ab_bench.sh base sra srb src st4 base sra srb src st4 2>&1 | tail -10
