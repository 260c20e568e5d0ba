#!/bin/bash
# secondary captures (under gpurun): FDM DST kernel (ncu --set full), launch lists of C3, C5fdm, C6
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
python bench.py --workload C5fdm --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/sp_fdm.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_dst" -s 2 -c 1 -o gpurun_out/prof_fdm \
    python bench.py --workload C5fdm --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/C5fdm_launches.csv \
    python bench.py --workload C5fdm --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/C3_launches.csv python tools/epoch_run.py C3 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/C6_launches.csv \
    python bench.py --workload C6 --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > /dev/null 2>&1
ls -la gpurun_out/
