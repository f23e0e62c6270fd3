mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamma.py -m gpu -q -x > gpurun_out/pytest_gamma.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gamma.log
timeout 300 python tools/e2e_breakdown.py 2>&1 | tail -3
