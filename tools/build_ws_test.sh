#!/bin/bash
# builds tools/ws_test (standalone check of k_gemm_ws.cu) for sm_100a
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Iinclude -o tools/ws_test tools/ws_test.cu -lcudart
