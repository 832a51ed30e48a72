# Round-2 final, 1 GPU (part 2): ncu --set full of one edge forward and one edge
# backward launch (the profile command exits 0 without ncu first).
set -x
B="python bench.py --steps 1 --warmup 2 --profile"
timeout 600 $B > gpurun_out/f11_plain.json 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_forward_kernel -s 12 -c 1 -o gpurun_out/f11_edge_fwd $B > gpurun_out/f11_ncu1.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_backward_kernel -s 9 -c 1 -o gpurun_out/f11_edge_bwd $B > gpurun_out/f11_ncu2.log 2>&1; echo rc=$?
ls -la gpurun_out/
