# backward / forward kernel phase counters at the bench shape (E=32, k=5, M=1) and E=24
set -x
timeout 600 python scripts/dbg_prof.py 32 > gpurun_out/prof2.log 2>&1; echo rc=$?
