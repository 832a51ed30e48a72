# timing ablation: forward e rows / e' stores with L2 evict_first
set -x
for v in "" fs; do
  tag=${v:-default}
  if [ -n "$v" ]; then export HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_exp$v.so; else unset HGNN_B200_LIB; fi
  for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ab_${tag}_$i.json 2>&1; echo rc=$?; done
done
