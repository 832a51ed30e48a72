# round-1 measurement pass: GPU tests, default bench, ncu launch list + full captures
timeout 900 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench_rc=$?
cat gpurun_out/bench_r1.json; tail -5 gpurun_out/bench_r1.err
B="python bench.py --steps 2 --warmup 3 --profile"
timeout 600 $B > gpurun_out/bench_prof_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward -s 2 -c 1 -o gpurun_out/prof_tc_bwd_c3 $B > gpurun_out/ncu_full_bwd.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_forward -s 4 -c 1 -o gpurun_out/prof_tc_fwd_c3 $B > gpurun_out/ncu_full_fwd.log 2>&1; echo ncu3_rc=$?
ls -la gpurun_out
