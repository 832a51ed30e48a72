set -x
timeout 600 python scripts/dbg_accuracy.py > gpurun_out/acc_rna.log 2>&1; echo rc=$?
HGNN_B200_LIB=paper_2410_01657_b200/lib/exp/libhgnn_b200_exptrunc.so timeout 600 python scripts/dbg_accuracy.py > gpurun_out/acc_trunc.log 2>&1; echo rc=$?
