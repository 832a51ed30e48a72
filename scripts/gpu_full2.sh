# full 1-GPU suite twice (reproducibility of a failure)
set -x
for i in 1 2; do timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/full2_$i.log 2>&1; echo rc=$?; tail -1 gpurun_out/full2_$i.log; done
