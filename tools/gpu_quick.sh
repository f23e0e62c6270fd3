mkdir -p gpurun_out
for v in default smemal smemal_t256 smemal_xv2; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 200 python bench.py --config c3 --steps 20 --warmup 2 --e2e-reps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac'], d['e2e']['matches_device_result'], d['b_norm'])"
done > gpurun_out/var.log 2>&1
cat gpurun_out/var.log
