mkdir -p gpurun_out
tail -1 gpurun_out/pytest_s1.log 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qb_sweep -c 2 -o gpurun_out/prof_qb python tools/time_qtilde.py c4 1 > gpurun_out/ncu_qb.log 2>&1; echo "ncu rc=$?"
