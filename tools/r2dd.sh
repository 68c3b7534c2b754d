mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hull or discrete or full_size or beyond_six or exact_settings or synthetic_scene or forward_matches" 2>&1 | tail -3
python tools/cmp_libs.py abvar/prev.so 2>&1 | tail -9 | head -8
bash tools/ab_bench.sh base prev base prev 2>&1 | tail -4
