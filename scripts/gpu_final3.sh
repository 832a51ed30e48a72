# final tree: smoke, full GPU suite, default bench line
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f7_smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f7_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/f7_bench.json 2> gpurun_out/f7_bench.err; echo bench_rc=$?
