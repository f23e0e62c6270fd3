#!/bin/bash
# build in-tree, then run a command on the GPU box:  tools/rg.sh TIMEOUT 'cmd'
cd /root/repo || exit 1
python -m paper_1503_08809_b200.build > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2" 2>&1 | grep -v "^\[gpurun\] sending"
