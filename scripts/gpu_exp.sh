# Quick A/B of a kernel change: parity tests, then two MP-stack bench lines (1 GPU).
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity_rc=$?
for i in 1 2; do timeout 600 python bench.py --no-e2e --no-train-step --no-cpu-baseline > gpurun_out/bench_exp.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_exp.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['ms_per_launch'], d['kernel_share']['node_bwd'])"; done
