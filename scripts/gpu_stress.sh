# stress: the in-process 8-rank a2a / na2a group cases 15x, then the full suite 2x
set -x
fails=0
for i in $(seq 1 15); do
  timeout 600 python -m pytest tests/test_gpu_local_group.py -q -x -k "test_group_matches_oracle" > gpurun_out/st_$i.log 2>&1 || { fails=$((fails+1)); cp gpurun_out/st_$i.log gpurun_out/st_fail_$i.log; }
done
echo "group loop failures: $fails"
for i in 1 2; do timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/st_full_$i.log 2>&1; echo rc=$?; tail -1 gpurun_out/st_full_$i.log; done
