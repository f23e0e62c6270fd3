#!/bin/bash
# Build a tuning variant of the library:  tools/build_variant.sh NAME -DMACRO=V ...
# Output: paper_1503_08809_b200/_native/variants/NAME.so (select with MG_LIB_PATH=...).
set -e
cd /root/repo/paper_1503_08809_b200/csrc
name=$1; shift
mkdir -p ../_native/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  --expt-relaxed-constexpr -Xcompiler -fPIC -shared "$@" -o ../_native/variants/$name.so \
  mg_api.cu mg_gamma.cu mg_qtilde.cu mg_gamma2d.cu
