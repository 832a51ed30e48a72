# GPU test suite + smoke + bench line (1 GPU)
set -x
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=12 > gpurun_out/r2h_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke_rc=$?
for f in 0 1; do
timeout 600 python bench.py --steps 3 --warmup 3 --profile --fact $f > gpurun_out/r2h_c3_f$f.json 2>&1; echo rc=$?
done
