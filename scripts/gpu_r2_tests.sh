# GPU test suite + smoke
set -x
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r2e_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-train-step > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench_rc=$?
