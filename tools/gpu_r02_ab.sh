#!/bin/bash
# round-2 call AB: DMMA form of the 2D cell sum (p <= 8) — parity, A/B against the per-cell
# kernel, ncu; the reference's 2D tests through the shim; NVTX ranges seen by ncu; small sizes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "Gamma2D" > gpurun_out/pytest_2d.log 2>&1; echo "2d tests rc=$?"
tail -5 gpurun_out/pytest_2d.log
timeout 600 python -m pytest tests/test_gpu_reference_suite.py -m gpu -q > gpurun_out/pytest_refsuite.log 2>&1; echo "ref suite rc=$?"
tail -3 gpurun_out/pytest_refsuite.log
rm -f gpurun_out/bench_2d_dmma.txt
for v in dmma lds; do
  if [ $v = dmma ]; then unset MG_G2D_LDS; else export MG_G2D_LDS=1; fi
  echo "== $v" >> gpurun_out/bench_2d_dmma.txt
  timeout 300 python tools/bench_2d.py >> gpurun_out/bench_2d_dmma.txt 2>&1
  timeout 300 python tools/bench_2d.py --lmax 256 --pmax 5 --r 300 --reps 2 >> gpurun_out/bench_2d_dmma.txt 2>&1
  timeout 300 python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 3 --no-ref >> gpurun_out/bench_2d_dmma.txt 2>&1
  timeout 300 python tools/bench_2d.py --lmax 1000 --pmax 6 --r 200 --reps 3 --no-ref >> gpurun_out/bench_2d_dmma.txt 2>&1
done
unset MG_G2D_LDS
cut -c1-330 gpurun_out/bench_2d_dmma.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ptable|k_gamma2d" -c 9 --csv \
    --log-file gpurun_out/launches_2d_dmma.csv python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 1 --no-ref > gpurun_out/ncu_2d_dmma.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gamma2d_dmma" -c 1 \
  -o gpurun_out/prof_2d_dmma python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 1 --no-ref > gpurun_out/ncu_2d_full.log 2>&1; echo "ncu full rc=$?"
# NVTX: only kernels inside the mg:gamma2d_cells range are profiled
timeout 600 ncu --nvtx --nvtx-include "mg:gamma2d_cells/" --metrics gpu__time_duration.sum --clock-control none -c 6 --csv \
    --log-file gpurun_out/launches_nvtx.csv python tools/bench_2d.py --reps 1 --no-ref > gpurun_out/ncu_nvtx.log 2>&1; echo "ncu nvtx rc=$?"
grep -c "k_gamma2d" gpurun_out/launches_nvtx.csv; grep -c "k_ptable" gpurun_out/launches_nvtx.csv
timeout 300 python tools/time_small.py > gpurun_out/time_small.txt 2>&1; cat gpurun_out/time_small.txt
