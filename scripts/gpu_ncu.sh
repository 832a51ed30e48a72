B="python bench.py --steps 2 --warmup 3 --profile"
timeout 600 $B > gpurun_out/bench_prof_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward -s 1 -c 1 -o gpurun_out/prof_edge_bwd_r1d $B > gpurun_out/ncu_full_bwd.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_forward -s 0 -c 1 -o gpurun_out/prof_edge_fwd_r1d $B > gpurun_out/ncu_full_fwd.log 2>&1; echo ncu3_rc=$?
du -sh gpurun_out
