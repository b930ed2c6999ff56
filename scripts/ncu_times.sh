# per-kernel durations (ncu, serialised) of three estimates of each workload (scripts/ncu_target.py)
for w in k25 lbm15 k7; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_times_$w.csv python scripts/ncu_target.py $w > /dev/null 2>&1
done
python scripts/ncu_times_sum.py gpurun_out/ncu_times_k25.csv gpurun_out/ncu_times_lbm15.csv gpurun_out/ncu_times_k7.csv
