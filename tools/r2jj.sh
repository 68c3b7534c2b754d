mkdir -p gpurun_out
python tools/cmp_libs.py abvar/norng.so 2>&1 | tail -9 | head -8
bash tools/ab_bench.sh base norng base norng 2>&1 | tail -4
B="bench.py --no-cpu-baseline --no-e2e --no-train --no-configs --steps 1 --warmup 0"
for v in base norng; do
  if [ $v = base ]; then unset CS_LIB_PATH; else export CS_LIB_PATH=abvar/$v.so; fi
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k "regex:forward_kernel" -s 2 -c 1 --csv --log-file gpurun_out/inst_$v.csv python $B > /dev/null 2>&1
  echo $v $(grep -v "^==" gpurun_out/inst_$v.csv | grep inst_executed | awk -F'","' '{print $NF}')
done
