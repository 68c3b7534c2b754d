# Build a variant of the library with extra nvcc flags on blend.cu/chain.cu:
#   bash tools/build_variant.sh <name> "-DFOO -DBAR"
# -> variants/<name>.so ; select it with CS_LIB_PATH=variants/<name>.so
set -e
name=$1; flags=$2
mkdir -p build/variants/$name variants
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
for f in blend chain; do nvcc $A $flags -c paper_2411_14974_b200/csrc/$f.cu -o build/variants/$name/$f.o; done
others=$(ls build/csrc/*.o | grep -v -e /blend.o -e /chain.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $others \
  build/variants/$name/blend.o build/variants/$name/chain.o -Xcompiler -fvisibility=hidden
