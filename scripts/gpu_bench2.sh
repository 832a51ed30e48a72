timeout 300 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_ts.json 2> gpurun_out/bench_ts.err; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_ts.json').readlines()[-1]); print(d['ms_per_step'], d['train_step'])"
tail -3 gpurun_out/bench_ts.err
