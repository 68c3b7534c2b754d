# build abvar/<name>.so: the current library with <file>.cu taken from git revision <rev>
# usage: bash tools/mkprev.sh <name> <rev> <file> [extra nvcc flags]
set -e
name=$1; rev=$2; f=$3; flags=$4
mkdir -p abvar build/ab_$name
git show $rev:paper_2411_14974_b200/csrc/$f.cu > build/ab_$name/$f.cu
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include -I paper_2411_14974_b200/csrc"
[ $f = preprocess ] && A="$A --fmad=false"
others=""
for o in build/csrc/*.o; do b=$(basename $o .o); [ "$b" != $f ] && others="$others $o"; done
nvcc $A $flags -c build/ab_$name/$f.cu -o build/ab_$name/$f.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abvar/$name.so $others build/ab_$name/$f.o -Xcompiler -fvisibility=hidden
