# ncu --set full captures of the HBM-bound kernels (aggregation, input-node adjoint gather)
# and the node-MLP kernels, one launch each (gpurun, 1 GPU). Reports in gpurun_out/.
B="python bench.py --steps 1 --warmup 3 --profile"
timeout 600 $B > gpurun_out/bench_prof_plain.log 2>&1; echo plain_rc=$?
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/prof_$1_r1h $B \
    > gpurun_out/ncu_$1.log 2>&1; echo $1_rc=$?
}
cap aggregate aggregate_kernel 0
cap dx_gather dx_gather_kernel 0
cap node_fwd mlp_tc_forward_kernel 1
cap node_bwd mlp_tc_backward_kernel 0
ls -la gpurun_out/*.ncu-rep
