# node-level adjoint with precomputed segment sums: parity + A/B timing
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_local_group.py -q -x > gpurun_out/ps_pytest.log 2>&1; echo rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ps_on_$i.json 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile --opt adjoint_presum=0 > gpurun_out/ps_off_$i.json 2>&1; echo rc=$?
done
