timeout 900 python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo bench_rc=$?
cat gpurun_out/bench_r1b.json; tail -3 gpurun_out/bench_r1b.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref_rc=$?
cat gpurun_out/bench_ref.json | tail -2
