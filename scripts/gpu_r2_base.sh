# round-2 baseline on the round-1 tree: GPU tests, bench line, edge-backward ncu capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench_rc=$?
B="python bench.py --steps 1 --warmup 3 --profile --elements 24"
timeout 300 $B > gpurun_out/r2a_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward -s 1 -c 1 -o gpurun_out/r2a_edge_bwd $B > gpurun_out/r2a_ncu.log 2>&1; echo ncu_rc=$?
