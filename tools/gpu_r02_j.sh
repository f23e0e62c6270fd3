#!/bin/bash
# round-2 call J: bounds-checked build over every pipeline kernel, p = 40 test, the
# multi-device + reference-suite files again, c2 and c4 bench lines
mkdir -p gpurun_out
MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/checked.so timeout 1500 python tools/checked_run.py > gpurun_out/j_checked.log 2>&1; echo "rc=$?" >> gpurun_out/j_checked.log
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "large_basis or MultiDevice" > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j_pytest.log
timeout 900 python bench.py --config c2 --steps 2 --warmup 1 --e2e-reps 1 --cpu-seconds 20 > gpurun_out/j_bench_c2.json 2> gpurun_out/j_bench_c2.err
timeout 2400 python bench.py --config c4 --steps 1 --warmup 1 --e2e-reps 1 --cpu-seconds 20 > gpurun_out/j_bench_c4.json 2> gpurun_out/j_bench_c4.err
tail -n 4 gpurun_out/j_checked.log; tail -n 4 gpurun_out/j_pytest.log
# diagnostic: K1/K2 time without their epilogue stores (MG_NO_EPI=1; results invalid, timing only)
VARS="default no_epi default" bash tools/var_run.sh > gpurun_out/j_noepi.log 2>&1
