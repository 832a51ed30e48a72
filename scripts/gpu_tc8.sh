timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 200 python scripts/dbg_prof.py
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'], d['kernel_share'], d['roofline']['ms_per_launch'])"
