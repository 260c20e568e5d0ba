#!/bin/bash
# per-kernel launch list of one bench step (under gpurun): tools/c4_breakdown.sh WORKLOAD TAG
W=${1:-C4}; TAG=${2:-x}
python bench.py --workload $W --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bd_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/bd_$TAG.csv python bench.py --workload $W --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bdn_$TAG.log 2>&1
tail -1 gpurun_out/bdn_$TAG.log
