mkdir -p gpurun_out
for v in 0 1 2 3; do
  export PMF_MID_VAR_FWD=$v PMF_MID_VAR_INV=$v PMF_MID_VAR_PSI=$v
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_plane_mid --csv --log-file gpurun_out/var_$v.csv python bench.py --workload C4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-time-update > gpurun_out/var_$v.log 2>&1
  python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-time-update > gpurun_out/varb_$v.json 2>&1
done
