set -x
for v in "" nolnb nostage notmem none; do
  tag=${v:-default}
  if [ -n "$v" ]; then export HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_exp$v.so; else unset HGNN_B200_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --profile --fact 0 > gpurun_out/pk_$tag.json 2>&1; echo rc=$?
done
unset HGNN_B200_LIB
timeout 600 python bench.py --steps 3 --warmup 3 --profile --fact 1 > gpurun_out/pk_fact1.json 2>&1; echo rc=$?
