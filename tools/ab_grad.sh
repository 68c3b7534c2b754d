# A/B the backward gradient error of library variants (variants/<name>.so) on the golden fixtures.
# usage: bash tools/ab_grad.sh base chain64 ...
for v in "$@"; do
  if [ $v = base ]; then unset CS_LIB_PATH; else export CS_LIB_PATH=variants/$v.so; fi
  echo "== $v"; python -m pytest tests/test_gpu_parity.py -q -k "backward_matches or synthetic" -s 2>&1 | grep "grad rel err"
done
