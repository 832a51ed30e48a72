# 2 GPUs of one box: NCCL multi-rank tests (consistency, C2, sequence guard), the
# weak-scaling N=2 bench line (halo exposed / raw shares), and configs[3]'s
# 64^3 / P=5 mesh split 2-way (memory-lean plan, ~99 M edges per GPU).
set -x
nvidia-smi --query-gpu=index,name,memory.total --format=csv
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/r2n2_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > gpurun_out/r2n2_bench.json 2> gpurun_out/r2n2_bench.err; echo bench_rc=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --scaling strong --elements 64 --steps 2 --warmup 3 --no-e2e --no-train-step \
  > gpurun_out/r2n2_c4.json 2> gpurun_out/r2n2_c4.err; echo c4_rc=$?
