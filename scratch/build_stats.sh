#!/bin/bash
# Builds a diagnostics copy of the library with pipeline wait counters.
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DDDF_PIPE_STATS=1 \
  paper_2306_16142_b200/csrc/ddf_api.cu -o scratch/statslib/libddf_b200.so
