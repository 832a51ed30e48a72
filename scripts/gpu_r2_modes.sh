# configs[4]: weak scaling (~4 M nodes per GPU) at N = 2 / 4 with the three halo
# modes (na2a = send/recv, a2a = padded all-to-all, none = inconsistent baseline)
set -x
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}"; }
for n in 2 4; do
  for m in na2a a2a none; do
    run $n 295$n$((${#m})) --mode $m --steps 3 --warmup 3 --no-e2e --no-train-step > gpurun_out/modes_${n}_$m.json 2> gpurun_out/modes_${n}_$m.err; echo rc=$?
  done
done
