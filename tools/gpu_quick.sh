mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gamma.py -m gpu -q -x 2>&1 | tail -1
for v in default prev default prev; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 600 python bench.py --no-cpu-baseline --e2e-reps 1 --steps 3 --warmup 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['roofline']['frac'],4), {k: round(v,1) for k,v in d['roofline']['kernel_ms_per_step'].items()})"
done
