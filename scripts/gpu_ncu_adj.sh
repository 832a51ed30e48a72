# ncu --set full of one node-level input-adjoint launch (factorised edge path)
set -x
B="python bench.py --steps 1 --warmup 2 --profile"
timeout 600 $B > gpurun_out/adj_plain.json 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_input_adjoint -s 4 -c 1 -o gpurun_out/adj $B > gpurun_out/adj_ncu.log 2>&1; echo rc=$?
