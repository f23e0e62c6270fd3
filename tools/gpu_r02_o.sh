#!/bin/bash
# round-2 call O: non-separable kernel variants (bisect the slow restructure; pipelined forms)
mkdir -p gpurun_out
for v in g2w16s2 a16g2 a16g4 a20g2 a20g1 a24g1 a24g2; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
  timeout 300 python bench.py --config c3 --steps 20 --no-cpu-baseline --e2e-reps 1 > gpurun_out/o_$v.json 2> gpurun_out/o_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/o_$v.json'));print('$v',round(d['ms_per_step'],3),round(d['roofline']['frac'],3),d['e2e'].get('matches_device_result'))" 2>&1 | tee -a gpurun_out/o_variants.txt
done
