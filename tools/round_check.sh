#!/bin/bash
# full GPU check under gpurun: tests, default bench line, C4 launch list (-> profiles/r2/launch_shares.json)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -5 gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('C4', d['value'], d['ms_per_step'], d['roofline']['frac'], d['time_update']['ms_per_step'], d['time_update']['hbm_frac'], d['e2e']['value'], d['cpu_baseline']['value'])
for k,v in d['also'].items(): print(k, v['value'], v['ms_per_step'], v['roofline']['frac'], (v['time_update'] or {}).get('ms_per_step'))"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/epoch_run.py C4 2 > /dev/null 2>&1
python tools/launch_breakdown.py gpurun_out/c4_launches.csv --last 7
