#!/bin/bash
# round-2 call Q: evidence with the final kernels — full GPU suite (with durations), smoke,
# default bench (c1), reference arm, c3, bounds-checked build, launch list, ncu of the N-split
# x contraction, c2 and c4 bench lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
( time timeout 1500 python -m pytest tests -m gpu -q --durations=15 ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
( time timeout 900 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
( time timeout 900 python bench.py --impl reference ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_c1_20.json 2> gpurun_out/bench_c1_20.err; echo "c1x20 rc=$?"
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/checked.so timeout 1500 python tools/checked_run.py > gpurun_out/checked.log 2>&1; echo "checked rc=$?"
tail -3 gpurun_out/checked.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 > gpurun_out/launches_c1.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_x_contract -c 1 -o gpurun_out/q_xns \
    python tools/prof_gamma.py --config c1 --l2 1400 1420 --reps 1 > gpurun_out/q_xns.log 2>&1; echo "ncu x rc=$?"
timeout 900 python bench.py --config c2 --steps 2 --warmup 1 --e2e-reps 1 --cpu-seconds 20 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 2400 python bench.py --config c4 --steps 1 --warmup 1 --e2e-reps 1 --cpu-seconds 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
