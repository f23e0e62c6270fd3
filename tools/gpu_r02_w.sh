#!/bin/bash
# round-2 call W: stage-1 k-tile of 128 (3-4 CTAs per SM) vs 256 (1-2 CTAs per SM)
mkdir -p gpurun_out; rm -f gpurun_out/qtilde_kt_ab.txt
for cfg in c1 c2 c4; do
  for v in default kt128a kt128b; do
    if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
    echo "== $cfg $v" >> gpurun_out/qtilde_kt_ab.txt
    timeout 300 python tools/time_qtilde.py $cfg 3 >> gpurun_out/qtilde_kt_ab.txt 2>&1
  done
done
unset MG_LIB_PATH
cat gpurun_out/qtilde_kt_ab.txt
for v in kt128a kt128b; do
MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so timeout 900 python -m pytest tests/test_gpu_stage1_nonsep.py -m gpu -q -k "Stage1 and (c0 or c1 or c2)" 2>&1 | tail -2
done
