#!/bin/bash
# usage: tools/build_variant.sh NAME "-DFLAG=.. -DFLAG2=.."   -> paper_2110_07663_b200/libsemlab_b200_NAME.so
# (A/B builds of k_space.cu; select at run time with SEMLAB_LIB=libsemlab_b200_NAME.so)
set -e
cd "$(dirname "$0")/.."
make -s -j8
NAME=$1; shift
mkdir -p build/var_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda \
  -Xcompiler -fPIC,-fopenmp -Ipaper_2110_07663_b200/csrc -Iinclude $* -c ${SRC:-paper_2110_07663_b200/csrc/k_space.cu} \
  -o build/var_$NAME/$(basename ${SRC:-k_space.cu}).o
objs=$(ls build/obj/*.o | grep -v $(basename ${SRC:-k_space.cu}).o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2110_07663_b200/libsemlab_b200_$NAME.so \
  $objs build/var_$NAME/$(basename ${SRC:-k_space.cu}).o -Xcompiler -fopenmp -L/usr/local/cuda/lib64 -lcusolver -lnccl -lgomp
