set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_group.py tests/test_gpu_configs.py -q -x > gpurun_out/ab_pytest.log 2>&1; echo pytest_rc=$?
for f in 0 1; do
timeout 600 python bench.py --steps 3 --warmup 3 --profile --fact $f > gpurun_out/ab_c3_f$f.json 2>&1; echo rc=$?
done
