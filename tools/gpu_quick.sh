mkdir -p gpurun_out
for v in default bk16 bk24 default bk16 bk24; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 600 python bench.py --no-cpu-baseline --e2e-reps 1 --steps 3 --warmup 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['roofline']['frac'],4), {k: round(v,1) for k,v in d['roofline']['kernel_ms_per_step'].items()})"
done
