# node-level adjoint with pipelined twin indices: parity + timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle or factorized or lean or tma or tensor_core" > gpurun_out/fb_pytest.log 2>&1; echo rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/fb_$i.json 2>&1; echo rc=$?; done
