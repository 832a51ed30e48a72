# factorised edge path timing on the final kernels (C3), 2 runs each
set -x
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --profile --fact 1 > gpurun_out/fact1_$i.json 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile --fact 0 > gpurun_out/fact0_$i.json 2>&1; echo rc=$?
done
