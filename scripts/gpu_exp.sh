set -x
for v in "" nopark; do
  tag=${v:-park}
  if [ -n "$v" ]; then export HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_exp$v.so; else unset HGNN_B200_LIB; fi
  for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/park_${tag}_$rep.json 2>&1; echo rc=$?
  done
done
