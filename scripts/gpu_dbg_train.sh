timeout 300 python scripts/dbg_train.py 16
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_train.csv python scripts/dbg_train.py 16 > /dev/null 2>&1; echo ncu_rc=$?
