# time variants of the library on a c1 slab (and optionally c4):  VARS="default v1" bash tools/var_run.sh
for v in ${VARS:-default}; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 200 python tools/time_slab.py --config c1 --l2 900 1300 --reps 3 2>&1 | tail -2
  if [ -n "$C4" ]; then timeout 300 python tools/time_slab.py --config c4 --l2 1500 1530 --reps 2 2>&1 | tail -2; fi
done
