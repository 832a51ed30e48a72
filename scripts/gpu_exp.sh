# reducer loop: one reducer (lib/exp) vs two, TMA on/off; parity of the fused forward
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle or factorized or tma or lean" > gpurun_out/red_pytest.log 2>&1; echo rc=$?
export HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_expr1.so
timeout 600 python bench.py --steps 3 --warmup 3 --profile --opt tma_gather=0 > gpurun_out/ab_r1.json 2>&1; echo rc=$?
unset HGNN_B200_LIB
timeout 600 python bench.py --steps 3 --warmup 3 --profile --opt tma_gather=0 > gpurun_out/ab_r2.json 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ab_tma.json 2>&1; echo rc=$?
