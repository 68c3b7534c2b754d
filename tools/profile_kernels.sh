# ncu --set full on one launch of each named kernel (separate captures), 1 GPU
for K in forward_kernel backward_kernel chain_kernel "onesweep_kernel<unsigned int>" duplicate_kernel; do
  tag=$(echo "$K" | tr -cd 'a-z_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -c 1 -o "gpurun_out/prof_$tag" \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "gpurun_out/prof_$tag.log" 2>&1
done
ls -la gpurun_out/*.ncu-rep
