#!/bin/bash
# K2 (x contraction) profiles at p=22 (c2) and p=30 (c4): plain run, then ncu --set full.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python tools/prof_gamma.py --config c2 --l2 1800 1805 --reps 2 > gpurun_out/k2_c2_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_x_contract -s 1 -c 1 \
    -o gpurun_out/k2_c2 python tools/prof_gamma.py --config c2 --l2 1800 1805 --reps 2 > gpurun_out/k2_c2_ncu.log 2>&1
python tools/prof_gamma.py --config c4 --l2 2000 2003 --reps 2 > gpurun_out/k2_c4_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_x_contract -s 1 -c 1 \
    -o gpurun_out/k2_c4 python tools/prof_gamma.py --config c4 --l2 2000 2003 --reps 2 > gpurun_out/k2_c4_ncu.log 2>&1
tail -3 gpurun_out/*.log
