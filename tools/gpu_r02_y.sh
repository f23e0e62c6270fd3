#!/bin/bash
# round-2 call Y: tiled 2D engine kernels (P table 64x64x32 register tiles, x-split cell kernel):
# parity, A/B against the first-cut kernels (variants/old2d.so), ncu of both kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "Gamma2D" > gpurun_out/pytest_2d.log 2>&1; echo "2d tests rc=$?"
tail -3 gpurun_out/pytest_2d.log
timeout 600 python -m pytest tests/test_gpu_reference_suite.py -m gpu -q > gpurun_out/pytest_refsuite.log 2>&1; echo "ref suite rc=$?"
tail -2 gpurun_out/pytest_refsuite.log
rm -f gpurun_out/bench_2d_ab.txt
for v in new old; do
  if [ $v = new ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/old2d.so; fi
  echo "== $v" >> gpurun_out/bench_2d_ab.txt
  timeout 300 python tools/bench_2d.py >> gpurun_out/bench_2d_ab.txt 2>&1
  timeout 300 python tools/bench_2d.py --lmax 256 --pmax 5 --r 300 --reps 2 >> gpurun_out/bench_2d_ab.txt 2>&1
  timeout 300 python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 3 --no-ref >> gpurun_out/bench_2d_ab.txt 2>&1
  timeout 300 python tools/bench_2d.py --lmax 1000 --pmax 6 --r 200 --reps 3 --no-ref >> gpurun_out/bench_2d_ab.txt 2>&1
done
unset MG_LIB_PATH
cat gpurun_out/bench_2d_ab.txt
for v in new old; do
  if [ $v = new ]; then unset MG_LIB_PATH; else export MG_LIB_PATH=paper_1503_08809_b200/_native/variants/old2d.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ptable|k_gamma2d" -c 12 --csv \
    --log-file gpurun_out/launches_2d_$v.csv python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 1 --no-ref > gpurun_out/ncu_2d_$v.log 2>&1; echo "ncu $v rc=$?"
done
unset MG_LIB_PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ptable|k_gamma2d_cells" -c 2 \
  -o gpurun_out/prof_2d python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 1 --no-ref > gpurun_out/ncu_2d_full.log 2>&1; echo "ncu full rc=$?"
