set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --elements 12 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo bench_small_rc=$?
tail -5 gpurun_out/bench_small.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench_rc=$?
tail -5 gpurun_out/bench_c3.log
