#!/bin/bash
# latency-bound configs under gpurun: all GPU tests, C1/C2/C3/C6 step medians (flushed, unflushed, predict), C6 warm launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
for w in C1 C2 C3 C6; do
python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --also "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['steps_timing']['median_ms'], d['steps_unflushed']['median_ms'], d['time_update']['ms_per_step'])"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum
ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/C6_warm.csv \
  python bench.py --workload C6 --steps 1 --warmup 3 --no-cpu --no-e2e --no-time-update --also "" > /dev/null 2>&1
python tools/launch_breakdown.py gpurun_out/C6_warm.csv --last 12
