#!/bin/bash
# round-2 call S: a = b pair fold A/B on the non-separable kernel (3 runs each, alternating)
mkdir -p gpurun_out
for i in 1 2 3; do
for v in default nofold; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
  timeout 300 python bench.py --config c3 --steps 30 --no-cpu-baseline --e2e-reps 1 > gpurun_out/s_$v.json 2> gpurun_out/s_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/s_$v.json'));print('$v',round(d['ms_per_step'],3),round(d['roofline']['frac'],3),d['e2e'].get('matches_device_result'))" 2>&1 | tee -a gpurun_out/s_variants.txt
done
done
