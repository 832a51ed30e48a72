# timing ablation: fused-forward reducer (64: no e' stores, 128: no reducer work)
set -x
for v in "" 64 128; do
  tag=${v:-default}
  if [ -n "$v" ]; then export HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_exp$v.so; else unset HGNN_B200_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ab_$tag.json 2>&1; echo rc=$?
done
