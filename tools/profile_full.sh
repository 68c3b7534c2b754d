# one ncu --set full capture of each hot kernel (first launch of each), 1 GPU
K='regex:preprocess_kernel|forward_kernel|backward_kernel|chain_kernel|onesweep_kernel|duplicate_kernel'
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c 7 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/prof_full.log 2>&1
ls -la gpurun_out/
