timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 200 python scripts/dbg_fwd.py
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-train-step 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'], d['kernel_share'], d['roofline']['ms_per_launch'], d['roofline']['frac'])"
