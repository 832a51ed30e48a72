# round-2 profiles at C3: bench line, ncu launch list of one step, --set full of
# the fused edge forward and the edge backward (one launch each)
set -x
B="python bench.py --steps 1 --warmup 3 --profile"
timeout 600 $B > gpurun_out/r2p_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 200 --csv --log-file gpurun_out/r2p_launches.csv $B > gpurun_out/r2p_ncu1.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_forward_kernel -s 12 -c 1 -o gpurun_out/r2p_edge_fwd $B > gpurun_out/r2p_ncu2.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward_kernel -s 9 -c 1 -o gpurun_out/r2p_edge_bwd $B > gpurun_out/r2p_ncu3.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dx_gather -s 5 -c 1 -o gpurun_out/r2p_dx_gather $B > gpurun_out/r2p_ncu4.log 2>&1; echo rc=$?
