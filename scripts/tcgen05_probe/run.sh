#!/bin/bash
# Build and run the tcgen05 DFT-64 probe (one B200): prints one JSON object per kernel.
set -e
D=$(cd "$(dirname "$0")" && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o "$D/tc_dft64" "$D/tc_dft64.cu"
timeout 120 "$D/tc_dft64" ${1:-1048576}
