#!/bin/bash
# round-2 call Z: 2D engine, second pass (P table at 2 CTAs per SM, 16 CTAs per SM of cell work)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "Gamma2D" > gpurun_out/pytest_2d.log 2>&1; echo "2d tests rc=$?"
tail -3 gpurun_out/pytest_2d.log
rm -f gpurun_out/bench_2d_v2.txt
timeout 300 python tools/bench_2d.py >> gpurun_out/bench_2d_v2.txt 2>&1
timeout 300 python tools/bench_2d.py --lmax 256 --pmax 5 --r 300 --reps 2 >> gpurun_out/bench_2d_v2.txt 2>&1
timeout 300 python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 3 --no-ref >> gpurun_out/bench_2d_v2.txt 2>&1
timeout 300 python tools/bench_2d.py --lmax 1000 --pmax 6 --r 200 --reps 3 --no-ref >> gpurun_out/bench_2d_v2.txt 2>&1
cat gpurun_out/bench_2d_v2.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ptable|k_gamma2d" -c 12 --csv \
    --log-file gpurun_out/launches_2d_v2.csv python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 1 --no-ref > gpurun_out/ncu_2d_v2.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ptable|k_gamma2d_cells" -c 2 \
  -o gpurun_out/prof_2d_v2 python tools/bench_2d.py --lmax 512 --pmax 8 --r 300 --reps 1 --no-ref > gpurun_out/ncu_2d_full.log 2>&1; echo "ncu full rc=$?"
