#!/bin/bash
# tools/variant.sh NAME "-DMACRO=V ..." — link a variant liblmfao_gpu.so (diagnostics; select it with LMFAO_LIB)
set -e
cd "$(dirname "$0")/.."
B=paper_1906_08687_b200/build
mkdir -p $B/var_$1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $2 -c paper_1906_08687_b200/csrc/cov.cu -o $B/var_$1/cov.cu.o
objs=$(ls $B/*.o | grep -v '/cov.cu.o')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/var_$1/lib.so $B/var_$1/cov.cu.o $objs -ldl -lcudart
echo $B/var_$1/lib.so
