# tcgen05 encoders: model-level tests + the default bench line (train step shares)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/enc_pytest.log 2>&1; echo rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/enc_c3.json 2> gpurun_out/enc_c3.err; echo rc=$?
