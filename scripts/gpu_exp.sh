set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/n128_pytest.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/n128_c3.json 2>&1; echo rc=$?
HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_expn64.so timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/n64_c3.json 2>&1; echo rc=$?
