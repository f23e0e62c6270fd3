# time non-separable kernel variants at config 3:  VARS="default ns_ch2_t512" bash tools/var_ns.sh
for v in ${VARS:-default}; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --e2e-reps 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],3), 'ms', round(r['frac'],4), 'match', d['e2e']['matches_device_result'], 'b_norm', d['b_norm'])"
done
