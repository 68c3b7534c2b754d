set -e
name=$1; flags=$2
mkdir -p build/variants/$name variants
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
nvcc $A $flags --fmad=false -c paper_2411_14974_b200/csrc/preprocess.cu -o build/variants/$name/preprocess.o
others=$(ls build/csrc/*.o | grep -v /preprocess.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so build/variants/$name/preprocess.o $others -Xcompiler -fvisibility=hidden
