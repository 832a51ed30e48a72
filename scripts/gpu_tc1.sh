timeout 300 python -m pytest tests/test_gpu_parity.py -k "tensor_core" -x -q > gpurun_out/tc1.log 2>&1; echo tc_rc=$?
tail -40 gpurun_out/tc1.log
