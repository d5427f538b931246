#!/bin/bash
# Build paper_1610_10061_b200/libpmedian_b200_<name>.so from the CURRENT csrc
# with extra nvcc flags for fitness.cu (K2 A/B switches, e.g. -DPMB_X_SPLITQ=0):
#   tools/build_variant.sh v1 "-DPMB_X_SPLITQ=0"
#   PMB_LIBRARY=paper_1610_10061_b200/libpmedian_b200_v1.so python tools/time_eval.py ...
set -e
name=$1; flags=$2
mkdir -p build_var/$name
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
nvcc $F -Xptxas --register-usage-level=10 $flags -c paper_1610_10061_b200/csrc/fitness.cu -o build_var/$name/fitness.o
others=$(ls build/*.o | grep -v '/fitness.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1610_10061_b200/libpmedian_b200_$name.so \
  $others build_var/$name/fitness.o -lcudart_static -lrt -ldl -lpthread
