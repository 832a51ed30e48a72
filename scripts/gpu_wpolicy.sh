# Edge-backward memory-policy experiments: parity tests, bench line, ncu captures of the edge and node backward.
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity_rc=$?; tail -2 gpurun_out/pytest_parity.log
timeout 600 python bench.py --no-e2e --no-train-step --no-cpu-baseline > gpurun_out/bench_wp.json 2> gpurun_out/bench_wp.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_wp.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['ms_per_launch'], d['kernel_share'], d['hbm_kernels'])"
B="python bench.py --steps 1 --warmup 3 --profile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward -s 1 -c 1 -o gpurun_out/prof_edge_bwd_r1x $B > gpurun_out/ncu_wp.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward -s 0 -c 1 -o gpurun_out/prof_node_bwd_r1x $B > gpurun_out/ncu_wp2.log 2>&1; echo ncu2_rc=$?
