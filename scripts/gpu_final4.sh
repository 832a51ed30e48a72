# final tree: smoke, full GPU suite, default bench line, 2 profile runs
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f8_smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f8_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/f8_pytest.log
timeout 900 python bench.py > gpurun_out/f8_bench.json 2> gpurun_out/f8_bench.err; echo bench_rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/f8_prof_$i.json 2>&1; echo rc=$?; done
