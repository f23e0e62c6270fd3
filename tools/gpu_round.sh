#!/bin/bash
# One GPU-box session for the round's evidence: parity tests, smoke, bench (+ reference arm,
# config 3), ncu launch list and a full ncu capture of the Γ contraction kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 > gpurun_out/b_small.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 300 python tools/prof_gamma.py > gpurun_out/prof_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(run|x|pair)_contract" -s 3 -c 3 \
      -o gpurun_out/prof_full python tools/prof_gamma.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_nonsep_warp -c 1 \
      -o gpurun_out/prof_nonsep python bench.py --config c3 --steps 1 --warmup 1 > gpurun_out/ncu_nonsep.log 2>&1; echo "ncu nonsep rc=$?"
fi
# multi-rank path on one GPU (gloo exchange; the real run uses NCCL, one GPU per rank)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 2 --steps 2 --warmup 1 --dist-backend gloo --e2e-reps 1 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank.err; echo "2-rank rc=$?"
# config 4 (p = 30) on one slab, extrapolated with the cost model
timeout 600 python tools/time_slab.py --config c4 --l2 1500 1530 --reps 2 > gpurun_out/c4_slab.log 2>&1; echo "c4 rc=$?"; tail -2 gpurun_out/c4_slab.log
