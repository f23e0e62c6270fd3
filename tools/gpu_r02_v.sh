#!/bin/bash
# round-2 call V: stage-1 sweeps with the chunk's Δ values prefetched: parity, timing A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_gamma.py -m gpu -q -k "Stage1 or Bessel or large_basis or end_to_end" > gpurun_out/pytest_s1.log 2>&1; echo "s1 rc=$?"
tail -3 gpurun_out/pytest_s1.log
rm -f gpurun_out/qtilde_prefetch_ab.txt
for cfg in c0 c1 c2 c4; do
  echo "== $cfg prefetch (default)" >> gpurun_out/qtilde_prefetch_ab.txt
  timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_prefetch_ab.txt 2>&1
  echo "== $cfg loads inside the recurrence loop (MG_QB_PREFETCH=0)" >> gpurun_out/qtilde_prefetch_ab.txt
  MG_LIB_PATH=paper_1503_08809_b200/_native/variants/noprefetch.so timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_prefetch_ab.txt 2>&1
done
cat gpurun_out/qtilde_prefetch_ab.txt
