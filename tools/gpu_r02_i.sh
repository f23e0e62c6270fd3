#!/bin/bash
# round-2 call I: full GPU test suite, smoke, the default bench line (c1), c3 with the full CPU
# restatement, the reference arm (c1), and the c1 launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/i_smi.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/i_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/i_bench_c1.json 2> gpurun_out/i_bench_c1.err
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --cpu-full > gpurun_out/i_bench_c3.json 2> gpurun_out/i_bench_c3.err
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/i_bench_ref_c1.json 2> gpurun_out/i_bench_ref_c1.err
tail -3 gpurun_out/i_pytest.log gpurun_out/i_smoke.log
