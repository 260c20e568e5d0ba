#!/bin/bash
# Latency-bound configs (C3, C6) under gpurun: warm-cache per-kernel launch list (ncu --cache-control none)
# and one --set full capture of each C3 plane kernel.  tools/lat_prof.sh [FULL=1]
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for w in C3 C6; do
  python tools/epoch_run.py $w 3 > gpurun_out/${w}_plain.log 2>&1 && \
  ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${w}_warm.csv python tools/epoch_run.py $w 3 > /dev/null 2>&1
  python tools/launch_breakdown.py gpurun_out/${w}_warm.csv --last 14 | tail -16
done
if [ "${1:-1}" = "1" ]; then
  ncu --set full --import-source on --clock-control none --cache-control none -k regex:"k_plane_(pre|fwd|mid|inv)" -s 4 -c 4 -o gpurun_out/prof_c3_full python tools/epoch_run.py C3 3 > /dev/null 2>&1
  ls -la gpurun_out/*.ncu-rep
fi
