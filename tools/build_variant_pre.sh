# build a variant with per-file flags including preprocess --fmad=false
set -e
name=$1; flags=$2
mkdir -p build/variants/$name variants
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
others=""
for o in build/csrc/*.o; do b=$(basename $o .o); [ "$b" != preprocess ] && others="$others $o"; done
nvcc $A --fmad=false $flags -c paper_2411_14974_b200/csrc/preprocess.cu -o build/variants/$name/preprocess.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $others build/variants/$name/preprocess.o -Xcompiler -fvisibility=hidden
