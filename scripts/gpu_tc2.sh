timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c3_tc.log 2>&1; echo bench_rc=$?
tail -2 gpurun_out/bench_c3_tc.log
B="python bench.py --steps 2 --warmup 1 --elements 12 --profile"
$B > gpurun_out/bench_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1_tc.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:mlp_tc_forward -s 0 -c 1 -o gpurun_out/prof_tc_fwd_r1 $B > gpurun_out/ncu_full_tc.log 2>&1; echo ncu2_rc=$?
