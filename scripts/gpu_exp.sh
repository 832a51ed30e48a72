set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor_core_backward or engine_matches_oracle or factorized or lean or deterministic" > gpurun_out/cs_pytest.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/cs_c3.json 2>&1; echo rc=$?
