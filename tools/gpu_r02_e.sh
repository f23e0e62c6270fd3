#!/bin/bash
# round-2 call E: staged (16 warps, l1 row from global) (TMA + LDS) non-separable DMMA kernel: parity, bench c3, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_parity_long.py::TestConfig3Full tests/test_gpu_parity_long.py::test_config3_resident_plan_matches_oneshot -m gpu -q -x > gpurun_out/e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e_pytest.log
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --e2e-reps 3 > gpurun_out/e_c3.json 2> gpurun_out/e_c3.err
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/e_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_nonsep_dmma -c 1 -o gpurun_out/e_nonsep_dmma \
    python bench.py --config c3 --steps 1 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/e_ncu.log 2>&1
tail -3 gpurun_out/e_pytest.log
