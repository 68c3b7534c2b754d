mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "discrete or full_size or synthetic or near_ties" 2>&1 | tail -1
python tools/cmp_libs.py abvar/prevs.so 2>&1 | tail -9 | head -7
bash tools/ab_bench.sh base prevs base prevs 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:tile_order|depth_fixup" --csv --log-file gpurun_out/to.csv python bench.py --no-cpu-baseline --no-e2e --no-train --no-configs --steps 1 --warmup 0 > /dev/null 2>&1; python tools/launches.py gpurun_out/to.csv
