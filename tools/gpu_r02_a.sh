#!/bin/bash
# round-2 call A: GPU tests (minus the c3 golden), x-tile A/B at p=22/30, one c2 Γ bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/a_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -k "not Config3Full" > gpurun_out/a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/a_pytest.log
for cfg in "c2 1200 1230 4" "c4 1500 1510 1"; do
  set -- $cfg
  echo "== $1 old tile MG_XTILE=$4" >> gpurun_out/a_xtile.log
  MG_XTILE=$4 timeout 600 python tools/time_slab.py --config $1 --l2 $2 $3 --reps 2 >> gpurun_out/a_xtile.log 2>&1
  echo "== $1 new default tile" >> gpurun_out/a_xtile.log
  timeout 600 python tools/time_slab.py --config $1 --l2 $2 $3 --reps 2 >> gpurun_out/a_xtile.log 2>&1
done
timeout 900 python bench.py --config c2 --steps 2 --warmup 1 --e2e-reps 1 --no-cpu-baseline > gpurun_out/a_bench_c2.json 2> gpurun_out/a_bench_c2.err
tail -5 gpurun_out/a_pytest.log
