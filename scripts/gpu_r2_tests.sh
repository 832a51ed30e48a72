# GPU test suite (incl. the new config-size and local-group tests) + smoke
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r2b_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo smoke_rc=$?
