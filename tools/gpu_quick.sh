mkdir -p gpurun_out
for v in default side2 side2b prev default side2 side2b prev; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  for sl in "300 420" "1500 1540"; do
    echo "== $v slab $sl"; timeout 200 python tools/time_slab.py --config c1 --l2 $sl --reps 3 2>&1 | tail -1
  done
done > gpurun_out/var.log 2>&1
cat gpurun_out/var.log
