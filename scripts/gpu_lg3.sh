# repeat the in-process group tests (flakiness check)
set -x
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_local_group.py -q -x > gpurun_out/lg3_$i.log 2>&1; echo rc=$?; tail -1 gpurun_out/lg3_$i.log; done
timeout 900 python -m pytest tests/test_gpu_local_group.py -q -x -k "8-4-2-32" > gpurun_out/lg3_k.log 2>&1; echo rc=$?; tail -1 gpurun_out/lg3_k.log
