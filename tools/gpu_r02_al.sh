#!/bin/bash
# round-2 call AL: 2D drop-in with the fingerprints hashed beside the GPU call
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamma.py tests/test_gpu_reference_suite.py -m gpu -q -k "Gamma2D or Engine2D or Acceptance or Harness" 2>&1 | tail -3
timeout 600 python bench.py --config 2d --steps 10 > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err; echo "2d rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_2d.json')); print(d['ms_per_step'], d['e2e'])"
timeout 300 python tools/bench_2d.py 2>&1 | cut -c1-300
timeout 300 python tools/bench_2d.py --lmax 256 --pmax 5 --r 300 --reps 2 2>&1 | cut -c1-300
