# Build a variant of the library with extra nvcc flags on some sources
# (default blend.cu chain.cu):
#   bash tools/build_variant.sh <name> "-DFOO -DBAR" ["sort blend"]
# -> variants/<name>.so ; select it with CS_LIB_PATH=variants/<name>.so
set -e
name=$1; flags=$2; files=${3:-blend chain}
mkdir -p build/variants/$name variants
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
others=""
for o in build/csrc/*.o; do
  b=$(basename $o .o); keep=1
  for f in $files; do [ "$b" = "$f" ] && keep=0; done
  [ $keep = 1 ] && others="$others $o"
done
for f in $files; do nvcc $A $flags -c paper_2411_14974_b200/csrc/$f.cu -o build/variants/$name/$f.o; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $others \
  $(for f in $files; do echo build/variants/$name/$f.o; done) -Xcompiler -fvisibility=hidden
