#!/bin/bash
# round-2 call M: non-separable kernel on the 6-register K order (NsSix) vs the rotation design
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_parity_long.py -m gpu -q --durations=12 > gpurun_out/pytest_ns.log 2>&1; echo "pytest rc=$?"
tail -20 gpurun_out/pytest_ns.log
timeout 600 python bench.py --config c3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3_six.json 2> gpurun_out/bench_c3_six.err; echo "c3 six rc=$?"
MG_LIB_PATH=paper_1503_08809_b200/_native/variants/rot8.so timeout 600 python bench.py --config c3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3_rot8.json 2> gpurun_out/bench_c3_rot8.err; echo "c3 rot8 rc=$?"
python - <<'P'
import json
for n in ("six","rot8"):
    try:
        d=json.load(open(f"gpurun_out/bench_c3_{n}.json")); print(n, d["ms_per_step"], d["roofline"]["frac"])
    except Exception as e: print(n, "failed", e)
P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nonsep_dmma -c 1 -o gpurun_out/m_nonsep_six \
    python bench.py --config c3 --steps 1 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/m_ncu.log 2>&1; echo "ncu rc=$?"
