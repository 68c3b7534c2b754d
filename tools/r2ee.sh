mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/build_variant.sh sl2k "-DCS_PROD_SLEEP_NS=2048" "blend" > /dev/null 2>&1
bash tools/build_variant.sh sl0 "-DCS_PROD_SLEEP_NS=0" "blend" > /dev/null 2>&1
bash tools/build_variant.sh sl8k "-DCS_PROD_SLEEP_NS=8192" "blend" > /dev/null 2>&1
bash tools/ab_bench.sh base sl2k sl0 sl8k base sl2k sl0 sl8k 2>&1 | tail -8
