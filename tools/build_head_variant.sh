#!/bin/bash
# Build the committed (HEAD) sources as a tuning variant: tools/build_head_variant.sh NAME [flags]
# Output: paper_1503_08809_b200/_native/variants/NAME.so (select with MG_LIB_PATH=...).
set -e
name=$1; shift
root=/root/repo
tmp=$(mktemp -d)
mkdir -p $tmp/paper_1503_08809_b200/csrc $tmp/include $root/paper_1503_08809_b200/_native/variants
for f in $(git -C $root ls-files paper_1503_08809_b200/csrc include); do git -C $root show HEAD:$f > $tmp/$f; done
cd $tmp/paper_1503_08809_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  --expt-relaxed-constexpr -Xcompiler -fPIC -shared "$@" \
  -o $root/paper_1503_08809_b200/_native/variants/$name.so mg_api.cu mg_gamma.cu mg_qtilde.cu mg_gamma2d.cu
rm -rf $tmp
