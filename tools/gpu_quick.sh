mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stage1_nonsep.py -m gpu -q -x > gpurun_out/pytest_nonsep.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_nonsep.log
timeout 300 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"; cat gpurun_out/bench_c3.json
