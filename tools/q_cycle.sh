#!/bin/bash
# quick cycle for the C4 path under gpurun: parity tests, event timings, ncu launch list
python -m pytest tests/test_gpu_plane.py -x -q -k "C4 or normalisation" 2>&1 | tail -3
python tools/epoch_run.py C4 4 > gpurun_out/er.log 2>&1; cat gpurun_out/er.log
python tools/epoch_run.py C4 4 --predict-only 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ql.csv python tools/epoch_run.py C4 2 > /dev/null 2>&1
python tools/launch_breakdown.py gpurun_out/ql.csv --last 7
