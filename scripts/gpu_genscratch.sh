# Encoder/decoder backward scratch discard: model tests, then the default bench line (train_step split).
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_model.log 2>&1; echo model_rc=$?; tail -2 gpurun_out/pytest_model.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['train_step']['ms_per_step'], d['train_step']['kernel_share'], d['train_step']['losses'])"
