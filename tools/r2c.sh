mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh chain64 "-DCS_ACC_F64 -DCS_CHAIN_F64" "blend chain capi" > /dev/null 2>&1
bash tools/build_variant.sh accurate "-DCS_ACC_F64 -DCS_CHAIN_F64 -DCS_BWD_ACCURATE -DCS_EXACT_RECIP -DCS_MAX_SHIFT" "blend chain capi" > /dev/null 2>&1
CS_LIB_PATH=variants/chain64.so timeout 900 python tools/grad_forced.py golden 2k 20k exact ortho 100k > gpurun_out/gf_chain64.txt 2>&1
CS_LIB_PATH=variants/accurate.so timeout 900 python tools/grad_forced.py golden 2k 20k exact ortho 100k > gpurun_out/gf_accurate.txt 2>&1
bash tools/ab_bench.sh chain64 accurate > gpurun_out/ab2.txt 2>&1
cat gpurun_out/ab2.txt
