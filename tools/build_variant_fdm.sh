#!/bin/bash
# variant of k_fdm.cu
set -e
cd /root/repo
NAME=$1; shift
mkdir -p build/var_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda \
  -Xcompiler -fPIC,-fopenmp -Ipaper_2110_07663_b200/csrc -Iinclude $* -c paper_2110_07663_b200/csrc/k_fdm.cu -o build/var_$NAME/k_fdm.cu.o
objs=$(ls build/obj/*.o | grep -v k_fdm.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2110_07663_b200/libsemlab_b200_$NAME.so \
  $objs build/var_$NAME/k_fdm.cu.o -Xcompiler -fopenmp -L/usr/local/cuda/lib64 -lcusolver -lnccl -lgomp
