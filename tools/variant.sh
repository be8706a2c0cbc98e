#!/bin/bash
# tools/variant.sh NAME SRC.cu "-DMACRO=V ..." — link a variant liblmfao_gpu.so in which SRC.cu (a file
# under csrc/, or any copy of one) replaces its namesake (diagnostics; select it with LMFAO_LIB)
set -e
cd "$(dirname "$0")/.."
B=paper_1906_08687_b200/build
mkdir -p $B/var_$1
base=$(basename $2)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Ipaper_1906_08687_b200/csrc $3 -c $2 -o $B/var_$1/$base.o
objs=$(ls $B/*.o | grep -v "/$base.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/var_$1/lib.so $B/var_$1/$base.o $objs -ldl -lcudart
echo $B/var_$1/lib.so
