# final tree: ncu launch list, then edge fwd / bwd captures
set -x
B="python bench.py --steps 1 --warmup 2 --profile"
timeout 600 $B > gpurun_out/f11_plain0.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f11_launches.csv $B > gpurun_out/f11_ncu0.log 2>&1; echo launches_rc=$?
bash scripts/gpu_r2_final2.sh
