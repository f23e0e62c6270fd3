#!/bin/bash
# round-2 call AD: final library (NVTX ranges, 2D engine kernels) -> full GPU suite, smoke,
# default bench, reference arm, config-3 bench, ncu launch list of the default bench command
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 > gpurun_out/b_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
cut -c1-300 gpurun_out/bench.json
