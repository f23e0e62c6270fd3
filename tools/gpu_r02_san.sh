#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call, only after a clean plain run of the same case:
#   bash tools/gpu_r02_san.sh racecheck|synccheck|memcheck|initcheck
TOOL=${1:-racecheck}
mkdir -p gpurun_out
export SAN_LMAX=${SAN_LMAX:-90}
timeout 600 python tools/sanitize_case.py > gpurun_out/san_plain_$TOOL.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 --log-file gpurun_out/san_$TOOL.txt \
    python tools/sanitize_case.py > gpurun_out/san_run_$TOOL.log 2>&1
echo "rc=$?" >> gpurun_out/san_run_$TOOL.log
tail -5 gpurun_out/san_$TOOL.txt gpurun_out/san_run_$TOOL.log
