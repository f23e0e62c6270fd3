for v in ${VARS:-default bk32st3}; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 200 python tools/time_slab.py --config c1 --l2 900 1300 --reps 3 2>&1 | tail -2
done
