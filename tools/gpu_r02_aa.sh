#!/bin/bash
# round-2 call AA: config 2 and config 4 bench lines with the final library and the contract's
# 3 warm-up steps (round-1 review: the c2/c4 lines had steps = 2 / 1)
mkdir -p gpurun_out
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --e2e-reps 1 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
cat gpurun_out/bench_c2.json | cut -c1-400
timeout 2700 python bench.py --config c4 --steps 2 --warmup 3 --e2e-reps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
cat gpurun_out/bench_c4.json | cut -c1-400
