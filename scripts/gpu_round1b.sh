set -x
timeout 900 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_gpu.log
B="python bench.py --steps 2 --warmup 1 --elements 12 --profile"
$B > gpurun_out/bench_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:mlp_backward -s 1 -c 1 -o gpurun_out/prof_edge_bwd_r1 $B > gpurun_out/ncu_full_bwd.log 2>&1; echo ncu2_rc=$?
ncu --set full --clock-control none --import-source on -k regex:mlp_forward -s 0 -c 1 -o gpurun_out/prof_edge_fwd_r1 $B > gpurun_out/ncu_full_fwd.log 2>&1; echo ncu3_rc=$?
ls -la gpurun_out
