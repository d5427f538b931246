#!/bin/bash
# Build paper_1610_10061_b200/libpmedian_b200_ab.so with csrc/fitness.cu taken
# from git revision $1 (default HEAD), for same-box A/B timing:
#   PMB_LIBRARY=paper_1610_10061_b200/libpmedian_b200_ab.so python tools/time_eval.py ...
set -e
rev=${1:-HEAD}
mkdir -p build_ab
git show "$rev":paper_1610_10061_b200/csrc/fitness.cu > paper_1610_10061_b200/csrc/fitness_ab.cu
trap 'rm -f paper_1610_10061_b200/csrc/fitness_ab.cu' EXIT
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
nvcc $F -Xptxas --register-usage-level=10 -c paper_1610_10061_b200/csrc/fitness_ab.cu -o build_ab/fitness.o
others=$(ls build/*.o | grep -v '/fitness.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1610_10061_b200/libpmedian_b200_ab.so \
  $others build_ab/fitness.o -lcudart_static -lrt -ldl -lpthread
