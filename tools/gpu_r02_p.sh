#!/bin/bash
# round-2 call P: final non-separable kernel (16 warps, groups of 2, NsSix): parity, bench, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_parity_long.py -m gpu -q -k "NonSeparable or Config3 or config3" > gpurun_out/pytest_ns.log 2>&1; echo "ns rc=$?"
tail -3 gpurun_out/pytest_ns.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --config c3 --steps 30 --cpu-full > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_c3.json'));print('c3',d['ms_per_step'],d['roofline']['frac'],d['e2e'],d['cpu_baseline'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nonsep_dmma -c 1 -o gpurun_out/p_nonsep \
    python bench.py --config c3 --steps 1 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/p_ncu.log 2>&1; echo "ncu rc=$?"
