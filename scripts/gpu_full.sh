# full 1-GPU test suite
set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/full_pytest.log 2>&1; echo rc=$?
