#!/bin/bash
# experiment builds of libglop (GLOP_LIB=... selects one at run time)
cd "$(dirname "$0")/../paper_1704_02278_b200/csrc"
for v in NOWORK NODRAIN; do
  nvcc -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 -shared -gencode arch=compute_100a,code=sm_100a \
    -I../../include -DGLOP_EXP_$v -o ../libglop_exp_$v.so glop.cu -lcudart &
done
wait
