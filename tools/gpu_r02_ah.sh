#!/bin/bash
# round-2 call AH: co-residency microbenchmark (tools/coresidency.cu)
mkdir -p gpurun_out; rm -f gpurun_out/coresidency.txt
for wa in 13 12 16; do for tb in 128 96 32 256; do for ord in 0 1; do
  timeout 60 tools/bin/coresidency $wa $tb $ord | tail -1 >> gpurun_out/coresidency.txt
done; done; done
cat gpurun_out/coresidency.txt
