set -x
./scripts/probe/tmem_shapes > gpurun_out/probe_tmem.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ldopt.json 2>&1; echo rc=$?
B="python bench.py --steps 1 --warmup 2 --profile"
timeout 600 $B > gpurun_out/r2p_plain2.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 56 -c 28 --csv --log-file gpurun_out/r2p_launches.csv $B > gpurun_out/r2p_ncu1.log 2>&1; echo rc=$?
