#!/bin/bash
# ptxas register/spill report of one csrc file: tools/ptxas_check.sh kernels_quad.cu [grep-pattern]
R=/root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Xptxas -v,-warn-spills -I $R/paper_2412_07240_b200/csrc -I $R/include -c $R/paper_2412_07240_b200/csrc/$1 -o /tmp/ptxas_check.o 2>&1 \
  | grep -E "error|spill|Used" | grep -E "error|${2:-.}"
