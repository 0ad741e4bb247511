#!/bin/bash
# tools/libcmsvd_prof.so: the library with k_eig.cu compiled under -DCMSVD_SYEV_PROF (phase cycles of k_syev_ql);
# needs the objects of a normal build (python -m paper_2601_11626_b200.build).
set -e
cd "$(dirname "$0")/../paper_2601_11626_b200"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I../include -DCMSVD_SYEV_PROF -c csrc/k_eig.cu -o /tmp/k_eig_prof.o
objs=$(ls build_obj/*.o | grep -v k_eig.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../tools/libcmsvd_prof.so $objs /tmp/k_eig_prof.o -lcudart
