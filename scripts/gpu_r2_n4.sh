# 4 GPUs of one box: the 4-rank NCCL tests, weak scaling N = 4 (configs[4]),
# strong scaling of configs[3]'s 64^3 / P=5 mesh at 4-way, and the E = 40 strong
# series at N = 1 / 2 / 4, all through bench.py (max over ranks, CUDA events).
set -x
nvidia-smi --query-gpu=index,name --format=csv
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/r2n4_pytest.log 2>&1; echo pytest_rc=$?
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}"; }
run 4 29521 --no-e2e > gpurun_out/r2n4_weak.json 2> gpurun_out/r2n4_weak.err; echo rc=$?
run 4 29522 --scaling strong --elements 64 --steps 2 --warmup 3 --no-e2e --no-train-step > gpurun_out/r2n4_c4.json 2> gpurun_out/r2n4_c4.err; echo rc=$?
for n in 2 4; do
  run $n 2953$n --scaling strong --steps 3 --warmup 3 --no-e2e --no-train-step > gpurun_out/r2n4_strong_$n.json 2> gpurun_out/r2n4_strong_$n.err; echo rc=$?
done
timeout 900 python bench.py --scaling strong --steps 3 --warmup 3 --no-e2e --no-train-step --no-cpu-baseline > gpurun_out/r2n4_strong_1.json 2> gpurun_out/r2n4_strong_1.err; echo rc=$?
