# Overlapped vs serial halo exchange (gpurun --gpus 2|4): 2-GPU tests, then a sweep of
# the SMs left to the exchange.  Lines in gpurun_out/overlap.jsonl.
OUT=gpurun_out/overlap.jsonl; : > $OUT
FLAGS="--steps 3 --warmup 3 --no-e2e --no-train-step --no-cpu-baseline"
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/pytest_n2.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_n2.log
run() {
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 $FLAGS ${@:2} >> $OUT 2>> gpurun_out/overlap.err
  echo "N=$1 ${@:2} rc=$?"
}
for n in 2 $([ "$NG" -ge 4 ] && echo 4); do
  run $n --scaling strong --halo-overlap 0
  for r in 0 1 2 4; do run $n --scaling strong --halo-overlap 1 --halo-sm-reserve $r; done
done
python - <<'PY'
import json
for l in open("gpurun_out/overlap.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); c = d["config"]
        print(d["n_gpus"], d["scaling"], c["mode"], c["elements_per_axis"], d.get("halo_overlap"), d.get("halo_sm_reserve"),
              round(d["ms_per_step"], 2), d["halo_share"], d["kernel_share"].get("edge_fwd"), d["kernel_share"].get("edge_bwd"))
PY
