#!/bin/bash
# round-2 call R: stage-1 sweeps with reciprocal-multiply recurrence steps: parity vs scipy, timing A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_gamma.py -m gpu -q -k "Stage1 or Bessel or large_basis or smoke or end_to_end" > gpurun_out/pytest_s1.log 2>&1; echo "s1 rc=$?"
tail -3 gpurun_out/pytest_s1.log
for cfg in c1 c4; do
  echo "== $cfg recip (default)" >> gpurun_out/qtilde_recip_ab.txt
  timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_recip_ab.txt 2>&1
  echo "== $cfg IEEE division per step (MG_QB_RECIP=0)" >> gpurun_out/qtilde_recip_ab.txt
  MG_LIB_PATH=paper_1503_08809_b200/_native/variants/norecip.so timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_recip_ab.txt 2>&1
done
cat gpurun_out/qtilde_recip_ab.txt
