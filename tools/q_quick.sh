#!/bin/bash
# quick C4 cycle: a few plane parity cases, event timings, ncu launch list of one epoch
python -m pytest tests/test_gpu_plane.py -x -q -k "C4_32x32x16x16 or C4_96x96x16x16 or C4_b3 or C3_32x32x16 or C3_128" 2>&1 | tail -2
bash tools/q_time.sh X=1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ql.csv python tools/epoch_run.py C4 2 > /dev/null 2>&1
python tools/launch_breakdown.py gpurun_out/ql.csv --last 6
