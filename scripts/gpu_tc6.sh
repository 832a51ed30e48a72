timeout 200 python scripts/dbg_grads.py 3 5 64 2 5
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 200 python scripts/dbg_prof.py
