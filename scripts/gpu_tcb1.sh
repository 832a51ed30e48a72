timeout 300 python -m pytest tests/test_gpu_parity.py -k "tensor_core_backward" -x -q > gpurun_out/tcb1.log 2>&1; echo rc=$?
tail -30 gpurun_out/tcb1.log
