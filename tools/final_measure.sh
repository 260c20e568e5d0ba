#!/bin/bash
# round-end measurement under gpurun: default bench line, reference arm, launch lists
# (C4, C5, C5fdm) and ncu --set full captures of the dominant kernels
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -2 gpurun_out/ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for w in C4 C5 C5fdm; do
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${w}_launches.csv python tools/epoch_run.py $w 2 > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"k_plane_fwd|k_q_mid|k_q_inv" -s 3 -c 3 -o gpurun_out/prof_c4_full python tools/epoch_run.py C4 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_resident_epoch" -s 1 -c 1 -o gpurun_out/prof_c5_full python tools/epoch_run.py C5 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
for w in C3; do
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${w}_launches.csv python tools/epoch_run.py $w 2 > /dev/null 2>&1
done
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/C6_launches.csv \
    python bench.py --workload C6 --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > /dev/null 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
