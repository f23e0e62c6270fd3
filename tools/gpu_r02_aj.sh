#!/bin/bash
# round-2 call AJ: DMMA form of the 2D cell sum with several M tiles (8 < p <= 24): parity and
# kernel time against the per-cell form (MG_G2D_LDS=1)
mkdir -p gpurun_out; rm -f gpurun_out/g2d_mtiles.txt
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "Gamma2D" 2>&1 | tail -3
for sz in "--lmax 96 --pmax 9 --r 100" "--lmax 96 --pmax 12 --r 100" "--lmax 96 --pmax 15 --r 60" "--lmax 64 --pmax 20 --r 40" "--lmax 64 --pmax 24 --r 24"; do
  for v in dmma lds; do
    if [ $v = dmma ]; then unset MG_G2D_LDS; else export MG_G2D_LDS=1; fi
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gamma2d_dmma|k_gamma2d_cells" -c 2 --csv \
      --log-file gpurun_out/l.csv python tools/bench_2d.py $sz --reps 1 --no-ref > gpurun_out/l.out 2>&1
    echo "$v | $sz | $(grep -o '"ns","[0-9]*"' gpurun_out/l.csv | tr '\n' ' ') | $(grep -o '"gpu_s": [0-9.e-]*' gpurun_out/l.out)" >> gpurun_out/g2d_mtiles.txt
  done
done
unset MG_G2D_LDS
cat gpurun_out/g2d_mtiles.txt
