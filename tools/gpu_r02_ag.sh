#!/bin/bash
# round-2 call AG: pair-product CTAs of 3 / 2 / 1 warps (can a side CTA be placed on the SM
# sub-partitions the 13-warp run contraction leaves room on?)
mkdir -p gpurun_out; rm -f gpurun_out/pp_threads_ab.txt
for v in default pp96 pp64 pp32 pp96u4; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== c1 $v" >> gpurun_out/pp_threads_ab.txt
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-reps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms_per_step'])" >> gpurun_out/pp_threads_ab.txt
done
unset MG_LIB_PATH
cat gpurun_out/pp_threads_ab.txt
