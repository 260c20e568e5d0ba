#!/bin/bash
# A/B timing of several builds of libpmf.so (under gpurun): tools/ab.sh WORKLOAD ROUNDS lib1.so lib2.so ...
# runs the same bench invocation with each library in turn, ROUNDS times; prints the step medians
W=${1:-C5}; R=${2:-3}; shift 2
for i in $(seq $R); do
  for L in "$@"; do
    PMF_LIB=$L python bench.py --workload $W --steps 20 --warmup 5 --no-cpu --no-e2e --also "" 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['steps_timing']['median_ms'], 4), round(d['time_update']['ms_per_step'], 4))"
  done
done
