# ncu --set full of one node-MLP backward launch (C3)
set -x
B="python bench.py --steps 1 --warmup 2 --profile"
timeout 600 $B > gpurun_out/nb_plain.json 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward_kernel -s 8 -c 1 -o gpurun_out/f6_node_bwd $B > gpurun_out/nb_ncu.log 2>&1; echo rc=$?
