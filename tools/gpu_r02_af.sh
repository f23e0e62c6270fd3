#!/bin/bash
# round-2 call AF: pair products released after the batch's panels (MG_SIDE=3) vs beside them
mkdir -p gpurun_out; rm -f gpurun_out/side3_ab.txt
for v in default side3 default side3; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== c1 $v" >> gpurun_out/side3_ab.txt
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-reps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms_per_step'])" >> gpurun_out/side3_ab.txt
done
for v in default side3; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== c2 $v" >> gpurun_out/side3_ab.txt
  timeout 900 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms_per_step'])" >> gpurun_out/side3_ab.txt
done
export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/side3.so
timeout 1200 python -m pytest tests/test_gpu_gamma.py tests/test_gpu_parity_long.py -m gpu -q -x -k "not Gamma2D and not nccl" 2>&1 | tail -3
unset MG_LIB_PATH
cat gpurun_out/side3_ab.txt
