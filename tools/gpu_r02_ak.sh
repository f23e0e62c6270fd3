#!/bin/bash
# round-2 call AK: final library -> full GPU suite, smoke, default bench, reference arm, c3 and
# 2d lines, ncu --set full of the three Γ contractions on a config-1 slab (round-2 traffic)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config 2d --steps 10 > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err; echo "2d rc=$?"
timeout 300 python tools/prof_gamma.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(run|x|pair)_contract" -s 3 -c 3 \
    -o gpurun_out/prof_full_r02 python tools/prof_gamma.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
cut -c1-300 gpurun_out/bench.json
