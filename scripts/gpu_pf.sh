# parity subset + C3 kernel times (2 runs) for a backward-kernel change
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_model.py -q -x -k "tensor_core_backward or engine_matches_oracle or factorized or lean or deterministic or model" > gpurun_out/pf_pytest.log 2>&1; echo rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/pf_c3_$i.json 2>&1; echo rc=$?; done
