mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh acc64 "-DCS_ACC_F64" "blend chain capi" > /dev/null 2>&1
timeout 900 python tools/grad_forced.py golden 2k 20k exact ortho k12 131k_tiles max_width 100k > gpurun_out/gf_base.txt 2>&1
CS_LIB_PATH=variants/acc64.so timeout 900 python tools/grad_forced.py golden 2k 20k exact ortho k12 131k_tiles max_width 100k > gpurun_out/gf_acc64.txt 2>&1
bash tools/ab_bench.sh base acc64 > gpurun_out/ab1.txt 2>&1
tail -3 gpurun_out/gf_base.txt gpurun_out/gf_acc64.txt; cat gpurun_out/ab1.txt
