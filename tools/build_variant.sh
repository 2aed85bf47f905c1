#!/bin/bash
# Dev: build variants/libseraph_<name>.so with extra nvcc defines for kernels.cu
# usage: bash tools/build_variant.sh <name> "-DFOO=1 -DBAR=0"
set -e
name=$1; defs=$2
mkdir -p variants build/var_$name
make -s lib >/dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1806_00762_b200/csrc $defs -c paper_1806_00762_b200/csrc/kernels.cu -o build/var_$name/kernels.o
objs=$(ls build/obj/*.o | grep -v '/kernels.o$')
g++ -o variants/libseraph_$name.so build/var_$name/kernels.o $objs -shared -L/usr/local/cuda/lib64 -lcudart -ldl -lpthread -Wl,-rpath,/usr/local/cuda/lib64
echo built variants/libseraph_$name.so
