#!/bin/bash
# round-2 call AI: final library -> full GPU suite, smoke, default bench, reference arm, 2d line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config 2d --steps 10 > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err; echo "2d rc=$?"
cut -c1-300 gpurun_out/bench.json
