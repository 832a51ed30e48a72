# node-level adjoint with 4 slots in flight: parity + timing, then the ncu captures of the final edge kernels
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/fa_pytest.log 2>&1; echo rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/fa_$i.json 2>&1; echo rc=$?; done
bash scripts/gpu_r2_final2.sh
