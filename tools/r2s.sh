mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant_pre.sh unr "-DCS_PRE_UNROLL_PROJ" > /dev/null 2>&1
bash tools/build_variant_pre.sh unr7 "-DCS_PRE_UNROLL_PROJ -DCS_PRE_BLOCKS=7" > /dev/null 2>&1
bash tools/build_variant_pre.sh unr5 "-DCS_PRE_UNROLL_PROJ -DCS_PRE_BLOCKS=5" > /dev/null 2>&1
CS_LIB_PATH=variants/unr.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "discrete or full_size or synthetic" 2>&1 | tail -1
bash tools/ab_bench.sh base unr unr7 unr5 base > gpurun_out/ab12.txt 2>&1; cat gpurun_out/ab12.txt
