#!/bin/bash
# round-2 call U: final library — full GPU suite, smoke, default bench, ncu of the stage-1 sweep (c4)
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q --durations=8 ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
( time timeout 900 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python tools/time_qtilde.py c4 1 > gpurun_out/u_qt.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qb_sweep -c 2 -o gpurun_out/u_qb \
    python tools/time_qtilde.py c4 1 > gpurun_out/u_ncu.log 2>&1; echo "ncu rc=$?"
