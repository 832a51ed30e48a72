timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tc3.log 2>&1; echo tc_rc=$?
tail -5 gpurun_out/tc3.log
B="python bench.py --steps 2 --warmup 1 --elements 12 --profile"
$B > gpurun_out/bench_prof_plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/bench_prof_plain.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_share'])"
ncu --set full --clock-control none --import-source on -k regex:mlp_tc_forward -s 0 -c 1 -o gpurun_out/prof_tc_fwd_r1b $B > gpurun_out/ncu_full_tc.log 2>&1; echo ncu2_rc=$?
