# Strong scaling (configs[3]) and halo-mode comparison (configs[4]) on a 4-GPU box:
#   gpurun --gpus 4 --timeout 3000 -- 'bash scripts/gpu_scaling.sh'
# One JSON line per run in gpurun_out/scaling.jsonl (MP-stack fwd+bwd only).
OUT=gpurun_out/scaling.jsonl; : > $OUT
FLAGS="--steps 3 --warmup 3 --no-e2e --no-train-step --no-cpu-baseline"
run() {  # run N extra-args...
  n=$1; shift
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --gpus 1 $FLAGS "$@" >> $OUT 2>> gpurun_out/scaling.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n $FLAGS "$@" >> $OUT 2>> gpurun_out/scaling.err
  fi
  echo "N=$n $* rc=$?"
}
for n in 1 2 4; do run $n --scaling strong; done
run 4 --scaling strong --elements 64
for m in a2a none; do for n in 2 4; do run $n --mode $m; done; done
python - <<'EOF'
import json
for l in open("gpurun_out/scaling.jsonl"):
    l = l.strip()
    if not l.startswith("{"):
        continue
    d = json.loads(l)
    c = d["config"]
    print(d["n_gpus"], d["scaling"], c["mode"], c["elements_per_axis"], round(d["ms_per_step"], 1),
          f"{d['value']:.3e}", d["halo_share"])
EOF
