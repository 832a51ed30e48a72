set -x
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_local_group.py -q -rs -s --durations=15 > gpurun_out/r2d_pytest.log 2>&1; echo pytest_rc=$?
