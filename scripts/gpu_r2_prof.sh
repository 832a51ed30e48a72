set -x
timeout 300 python scripts/dbg_prof.py 24 1 > gpurun_out/r2f_prof_fact.log 2>&1; echo rc=$?
timeout 300 python scripts/dbg_prof.py 24 0 > gpurun_out/r2f_prof_nofact.log 2>&1; echo rc=$?
B="python bench.py --steps 1 --warmup 3 --profile --elements 24"
timeout 300 $B > gpurun_out/r2f_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward_kernel -s 1 -c 1 -o gpurun_out/r2f_edge_bwd $B > gpurun_out/r2f_ncu.log 2>&1; echo ncu_rc=$?
