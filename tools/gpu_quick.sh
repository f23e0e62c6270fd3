mkdir -p gpurun_out
for v in default x13 default x13; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== c4 $v"; timeout 600 python tools/time_slab.py --config c4 --l2 1500 1530 --reps 2 2>&1 | tail -1
done
