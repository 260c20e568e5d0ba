#!/bin/bash
# One GPU iteration (run under gpurun): gpu tests, bench, ncu capture of the top kernel.
#   tools/gpu_cycle.sh TAG [TESTS=1] [NCU=1] [KREGEX=k_resident_epoch] [BENCHARGS=""]
TAG=${1:-x}; TESTS=${2:-1}; NCU=${3:-1}; KRE=${4:-k_resident_epoch}; BARGS=${5:-}
mkdir -p gpurun_out
if [ "$TESTS" = "1" ]; then python -m pytest tests -q -m gpu 2>&1 | tail -3; fi
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-time-update $BARGS > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cut -c1-260 gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
if [ "$NCU" = "1" ]; then
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-time-update $BARGS > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/prof_$TAG \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-time-update $BARGS > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi
