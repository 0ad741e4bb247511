#!/bin/bash
# Build the standalone eigenvalue-kernel microbenchmark (tools/eigbench.cu).
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I../include -Xptxas -v "$@" -o eigbench_w8 eigbench.cu 2>&1 | grep -E "error|k_tridiag|k_bisect" -A2 | grep -E "error|Used|spill" || true
