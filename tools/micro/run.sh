#!/bin/bash
# builds and runs the microbenchmarks on the GPU box; JSON to gpurun_out/
set -e
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I ../../paper_2412_07240_b200/csrc"
for b in "$@"; do
  $NV -o /tmp/$b $b.cu
  timeout 120 /tmp/$b > ../../gpurun_out/$b.json
  cat ../../gpurun_out/$b.json
done
