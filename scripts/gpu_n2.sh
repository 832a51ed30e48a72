timeout 600 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/pytest_n2.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench_rc=$?
tail -1 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
