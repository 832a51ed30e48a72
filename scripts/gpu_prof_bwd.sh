B="python bench.py --steps 1 --warmup 1 --elements 8 --profile"
$B > gpurun_out/bench_prof_plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward -s 1 -c 1 -o gpurun_out/prof_tc_bwd_r1 $B > gpurun_out/ncu_full_tcb.log 2>&1; echo ncu_rc=$?
