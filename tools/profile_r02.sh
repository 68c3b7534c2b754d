# Round-2 profiles: launch list of one frame + ncu --set full of one launch per hot kernel.
# usage: bash tools/profile_r02.sh <tag> [kernel[:skip] ...]
tag=${1:-r02}; shift
KS=("$@")
[ ${#KS[@]} -eq 0 ] && KS=(forward_kernel backward_kernel preprocess_kernel chain_kernel onesweep_kernel:8 duplicate_scan_kernel)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="bench.py --no-cpu-baseline --no-e2e --no-train --no-configs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python $B --steps 2 --warmup 1 > gpurun_out/${tag}_launches.log 2>&1
for KK in "${KS[@]}"; do
  K=${KK%%:*}; S=0; [ "$KK" != "$K" ] && S=${KK##*:}
  k=$(echo "$K" | tr -cd 'a-z_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c 1 -o "gpurun_out/${tag}_prof_$k" \
      python $B --steps 1 --warmup 0 > "gpurun_out/${tag}_prof_$k.log" 2>&1
done
ls -la gpurun_out/*.ncu-rep
