#!/bin/bash
# event timings of the C4 epoch and predict under variants (env settings as args)
for v in "$@"; do
  echo "== $v"
  env $v python tools/epoch_run.py C4 4 2>&1 | tail -2
  env $v python tools/epoch_run.py C4 4 --predict-only 2>&1 | tail -1
done
