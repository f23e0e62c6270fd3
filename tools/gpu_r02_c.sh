#!/bin/bash
# round-2 call C: DMMA instruction counts of the three contractions (c1 slab, p = 15) next to
# the plan's executed-FLOP formula, plus the full-step launch list of the c1 bench.
mkdir -p gpurun_out
python tools/prof_gamma.py --config c1 --l2 1400 1420 --reps 1 > gpurun_out/c_plain.log 2>&1 && \
ncu --metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__ops_path_tensor_src_fp64.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"k_run_contract|k_x_contract|k_pair_contract" --csv \
    --log-file gpurun_out/c_dmma_counts.csv python tools/prof_gamma.py --config c1 --l2 1400 1420 --reps 1 > gpurun_out/c_ncu.log 2>&1
for cfg in c2 c4; do
  python tools/prof_gamma.py --config $cfg --l2 1500 1503 --reps 1 > gpurun_out/c_plain_$cfg.log 2>&1 && \
  ncu --metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:"k_run_contract|k_x_contract|k_pair_contract" --csv \
      --log-file gpurun_out/c_dmma_counts_$cfg.csv python tools/prof_gamma.py --config $cfg --l2 1500 1503 --reps 1 > gpurun_out/c_ncu_$cfg.log 2>&1
done
ls -la gpurun_out
