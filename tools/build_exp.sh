#!/bin/bash
# experiment build of libglop: tools/build_exp.sh NAME "-DFOO -DBAR" -> paper_1704_02278_b200/libglop_exp_NAME.so
# (select at run time with GLOP_LIB=$PWD/paper_1704_02278_b200/libglop_exp_NAME.so)
cd "$(dirname "$0")/../paper_1704_02278_b200/csrc"
nvcc -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 -shared -gencode arch=compute_100a,code=sm_100a \
  -I../../include $2 -o ../libglop_exp_$1.so glop.cu hostcopy.cpp -lcudart
