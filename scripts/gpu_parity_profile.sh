timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 200 python scripts/dbg_prof.py
