#!/bin/bash
# round-2 call X (re-entry): rebuilt library on a fresh container -> full GPU suite, smoke,
# default bench, reference arm, 2D engine timing (before its kernel rewrite)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python tools/bench_2d.py > gpurun_out/bench_2d_before.json 2> gpurun_out/bench_2d.err; echo "2d rc=$?"
timeout 600 python tools/bench_2d.py --lmax 256 --pmax 5 --r 300 --reps 2 >> gpurun_out/bench_2d_before.json 2>> gpurun_out/bench_2d.err; echo "2d rc=$?"
cat gpurun_out/bench.json gpurun_out/bench_2d_before.json
