#!/bin/bash
# C3 check under gpurun: plane/full-size/eigen-grid GPU tests, C3 bench steps, warm-cache launch list
mkdir -p gpurun_out
python -m pytest tests/test_gpu_plane.py tests/test_gpu_fullsize.py tests/test_gpu_eigen_grid.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
python bench.py --workload C3 --steps 20 --warmup 5 --no-cpu --no-e2e --also "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['steps_timing']['median_ms'], d['steps_unflushed']['median_ms'], d['time_update']['ms_per_step'])"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active
ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/C3_warm3.csv python tools/epoch_run.py C3 3 > /dev/null 2>&1
python tools/launch_breakdown.py gpurun_out/C3_warm3.csv --last 6
