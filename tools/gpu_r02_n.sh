#!/bin/bash
# round-2 call N: non-separable stage body (full/tail paths, no proxy fence, pointer cursor);
# N-split x tiles at p = 22 / 30; every-tile parity test
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -k "every_x_contraction_tile" > gpurun_out/pytest_tiles.log 2>&1; echo "tiles rc=$?"
tail -5 gpurun_out/pytest_tiles.log
timeout 900 python -m pytest tests/test_gpu_stage1_nonsep.py tests/test_gpu_parity_long.py -m gpu -q -k "NonSeparable or Config3 or config3" > gpurun_out/pytest_ns.log 2>&1; echo "ns rc=$?"
tail -3 gpurun_out/pytest_ns.log
timeout 600 python bench.py --config c3 --steps 30 --no-cpu-baseline > gpurun_out/bench_c3_n.json 2> gpurun_out/bench_c3_n.err; echo "c3 rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_c3_n.json'));print('c3',d['ms_per_step'],d['roofline']['frac'])"
run() { echo "== $1 MG_XTILE=$4" >> gpurun_out/xtile_ns2_ab.txt; MG_XTILE=$4 timeout 600 python tools/time_slab.py --config $1 --l2 $2 $3 --reps 3 >> gpurun_out/xtile_ns2_ab.txt 2>&1; }
run c1 1400 1440 5
run c2 1500 1530 2
run c2 1500 1530 6
run c4 1500 1510 3
run c4 1500 1510 7
cat gpurun_out/xtile_ns2_ab.txt
