mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
python bench.py --workload C3 --steps 20 --warmup 5 --no-cpu --no-e2e --also "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['steps_timing']['median_ms'], d['steps_unflushed']['median_ms'], d['time_update']['ms_per_step'])"
bash tools/c6prof.sh
