mkdir -p gpurun_out
for v in default qxt1 qxt2; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/$v.so; fi
  echo "== $v"; timeout 300 python tools/time_qtilde.py c1 3 2>&1 | tail -1; timeout 300 python tools/time_qtilde.py c4 2 2>&1 | tail -1
done
