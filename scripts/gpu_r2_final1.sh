# Round-2 final, 1 GPU (part 1): smoke, full GPU suite, default bench line,
# reference arm, ncu launch list of the profile command.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f4_smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/f4_ref.json 2> gpurun_out/f4_ref.err; echo ref_rc=$?
B="python bench.py --steps 1 --warmup 2 --profile"
timeout 600 $B > gpurun_out/f4_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f4_launches.csv $B > gpurun_out/f4_ncu0.log 2>&1; echo launches_rc=$?
