# TMA-gathered fused edge forward: prefetched producer indices
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tma" > gpurun_out/tma_pytest.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/tma_on.json 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile --opt tma_gather=0 > gpurun_out/tma_off.json 2>&1; echo rc=$?
