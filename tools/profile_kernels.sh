# ncu --set full on one launch of each named kernel (separate captures), 1 GPU,
# plus the launch list (gpu__time_duration per launch) of a short bench run.
# usage: bash tools/profile_kernels.sh <tag> [kernel[:skip] ...]
tag=${1:-r01}; shift
KS=("$@")
[ ${#KS[@]} -eq 0 ] && KS=(preprocess_kernel forward_kernel backward_kernel chain_kernel onesweep_kernel:8 duplicate_kernel)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train > gpurun_out/${tag}_launches.log 2>&1
for KK in "${KS[@]}"; do
  K=${KK%%:*}; S=0; [ "$KK" != "$K" ] && S=${KK##*:}
  k=$(echo "$K" | tr -cd 'a-z_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c 1 -o "gpurun_out/${tag}_prof_$k" \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-train > "gpurun_out/${tag}_prof_$k.log" 2>&1
done
ls -la gpurun_out/*.ncu-rep
