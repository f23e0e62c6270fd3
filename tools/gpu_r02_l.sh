#!/bin/bash
# round-2 call L: N-split x-contraction tile (p = 15) A/B on a c1 slab, p = 15 parity tests, durations
mkdir -p gpurun_out
for xt in 0 5; do
  echo "== c1 MG_XTILE=$xt" >> gpurun_out/xtile_ns_ab.txt
  MG_XTILE=$xt timeout 600 python tools/time_slab.py --config c1 --l2 1400 1440 --reps 3 >> gpurun_out/xtile_ns_ab.txt 2>&1
done
echo "== c1 default" >> gpurun_out/xtile_ns_ab.txt
timeout 600 python tools/time_slab.py --config c1 --l2 1400 1440 --reps 3 >> gpurun_out/xtile_ns_ab.txt 2>&1
cat gpurun_out/xtile_ns_ab.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=40 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -60 gpurun_out/pytest_gpu.log
