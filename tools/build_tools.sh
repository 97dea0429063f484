#!/bin/bash
# Build the stand-alone microbenchmarks/probes next to their sources (binaries are not committed).
set -e
cd "$(dirname "$0")"
for t in fp64_peak probe_mix_bw umma_i8_test; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o $t $t.cu
done
