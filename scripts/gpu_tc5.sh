timeout 300 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/tc5.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/tc5.log
timeout 200 python scripts/dbg_prof.py
