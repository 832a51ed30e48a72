# timing ablation: backward weight ring depth 1 with staging ring 4 / 5
set -x
for v in "" w1s4 w1s5; do
  tag=${v:-default}
  if [ -n "$v" ]; then export HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_exp$v.so; else unset HGNN_B200_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ab_$tag.json 2>&1; echo rc=$?
done
