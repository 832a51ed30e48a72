# ncu launch list of the bench command (per-kernel share of the step), 1 GPU.
B="python bench.py --steps 2 --warmup 3 --profile"
timeout 600 $B > gpurun_out/bench_prof_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
