#!/bin/bash
# round-2 call B: non-separable DMMA kernel (tests, A/B vs DFMA, bench c3 with CPU check),
# c3 golden tests, reference suite through the drop-in, multi-device tests, then ncu of the
# DMMA kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_parity_long.py::TestConfig3Full tests/test_gpu_parity_long.py::test_config3_resident_plan_matches_oneshot tests/test_gpu_reference_suite.py "tests/test_gpu_gamma.py::TestMultiDevice" -m gpu -q > gpurun_out/b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b_pytest.log
MG_NS_DFMA=1 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --e2e-reps 2 --no-cpu-baseline > gpurun_out/b_c3_dfma.json 2> gpurun_out/b_c3_dfma.err
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --e2e-reps 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/b_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_nonsep_dmma -c 1 -o gpurun_out/b_nonsep_dmma \
    python bench.py --config c3 --steps 1 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
tail -3 gpurun_out/b_pytest.log
