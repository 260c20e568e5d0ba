#!/bin/bash
# ncu --set full of the first epoch's plane-path kernels matching REGEX (under gpurun):
#   tools/prof_plane.sh WORKLOAD TAG REGEX [COUNT]
W=${1:-C4}; TAG=${2:-x}; RE=${3:-k_plane}; CNT=${4:-3}
mkdir -p gpurun_out
python bench.py --workload $W --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > gpurun_out/pp_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$RE" -c $CNT -o gpurun_out/prof_$TAG \
    python bench.py --workload $W --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > gpurun_out/ppn_$TAG.log 2>&1
tail -1 gpurun_out/ppn_$TAG.log
