#!/bin/bash
# round-2 call AC: warp count / fragments per warp / chunk size of the DMMA 2D cell kernel
mkdir -p gpurun_out; rm -f gpurun_out/g2d_variants.txt
timeout 600 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "Gamma2D" 2>&1 | tail -2
for v in default w8f3k64 w8f3k128 w12f2k128 w16f2k64 w16f2k128; do
  if [ $v = default ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/$v.so; fi
  for sz in "--lmax 512 --pmax 8 --r 300" "--lmax 1000 --pmax 6 --r 200" "--lmax 256 --pmax 5 --r 300"; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gamma2d_dmma" -c 3 --csv \
      --log-file gpurun_out/l.csv python tools/bench_2d.py $sz --reps 2 --no-ref > /dev/null 2>&1
    echo "$v | $sz | $(grep -o '"ns","[0-9]*"' gpurun_out/l.csv | tr '\n' ' ')" >> gpurun_out/g2d_variants.txt
  done
done
unset MG_LIB_PATH
cat gpurun_out/g2d_variants.txt
