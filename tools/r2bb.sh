python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant_pre.sh shl1 "-DCS_PRE_SH_L1" > /dev/null 2>&1
bash tools/build_variant_pre.sh shl1ph "-DCS_PRE_SH_L1 -DCS_PRE_PHASES" > /dev/null 2>&1
CS_LIB_PATH=variants/shl1ph.so python tools/pre_phases.py
bash tools/ab_bench.sh base shl1 base shl1 2>&1 | tail -4
