mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant_pre.sh nofast "-DCS_NO_HULL_FAST" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hull or discrete or full_size or beyond_six or exact_settings or synthetic_scene" 2>&1 | tail -3
python tools/cmp_libs.py variants/nofast.so 2>&1 | tail -9 | head -8
bash tools/ab_bench.sh base nofast base nofast 2>&1 | tail -4
