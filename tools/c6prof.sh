#!/bin/bash
# C6 (pencil, terrain/GM) under gpurun: warm-cache launch list of one bench step and ncu --set full of its kernels
mkdir -p gpurun_out
python bench.py --workload C6 --steps 20 --warmup 5 --no-cpu --no-e2e --also "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C6', d['steps_timing']['median_ms'], d['steps_unflushed']['median_ms'], d['time_update']['ms_per_step'])"
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/C6_warm.csv \
  python bench.py --workload C6 --steps 1 --warmup 3 --no-cpu --no-e2e --no-time-update --also "" > /dev/null 2>&1
python tools/launch_breakdown.py gpurun_out/C6_warm.csv --last 12
ncu --set full --import-source on --clock-control none --cache-control none -k "regex:k_points|k_axis0_r2c|k_regrid_rows" -s 3 -c 3 -o gpurun_out/prof_c6 \
  python bench.py --workload C6 --steps 1 --warmup 3 --no-cpu --no-e2e --no-time-update --also "" > gpurun_out/c6ncu.log 2>&1
tail -2 gpurun_out/c6ncu.log; ls -la gpurun_out/prof_c6.ncu-rep
