# Final round check on a 4-GPU box (gpurun --gpus 4): smoke, full GPU suite (2- and 4-rank
# tests included), default 1-GPU bench line, 2- and 4-GPU weak-scaling lines.
bash scripts/gpu_check.sh
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/pytest_multirank.log 2>&1; echo multirank_rc=$?; tail -3 gpurun_out/pytest_multirank.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
    bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo bench_n${n}_rc=$?
  tail -1 gpurun_out/bench_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['value'], d['e2e']['value'], d['halo_share'], d['config']['workload'])"
done
