mkdir -p gpurun_out
CS_LIB_PATH=abvar/anch.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "backward or grad or chain" 2>&1 | tail -2
bash tools/ab_bench.sh base prevb anch sl0 base prevb anch sl0 2>&1 | tail -8
