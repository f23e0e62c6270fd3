#!/bin/bash
# round-2 call AE: bench.py --config 2d, new 2D tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "Gamma2D" 2>&1 | tail -3
timeout 600 python bench.py --config 2d --steps 10 > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err; echo "2d bench rc=$?"
cat gpurun_out/bench_2d.json; tail -3 gpurun_out/bench_2d.err
