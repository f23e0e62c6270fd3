#!/bin/bash
# round-2 call T: stage-1 sweeps skipping dead (k tile, chunk) pairs: parity vs scipy, timing A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_gamma.py -m gpu -q -k "Stage1 or Bessel or large_basis or end_to_end" > gpurun_out/pytest_s1.log 2>&1; echo "s1 rc=$?"
tail -3 gpurun_out/pytest_s1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
rm -f gpurun_out/qtilde_skip_ab.txt
for cfg in c1 c2 c4; do
  echo "== $cfg skip (default)" >> gpurun_out/qtilde_skip_ab.txt
  timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_skip_ab.txt 2>&1
  echo "== $cfg every (k tile, chunk) pair (MG_QB_SKIP=0)" >> gpurun_out/qtilde_skip_ab.txt
  MG_LIB_PATH=paper_1503_08809_b200/_native/variants/noskip.so timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_skip_ab.txt 2>&1
done
cat gpurun_out/qtilde_skip_ab.txt
