#!/bin/bash
# Build tuning variants of the library: tools/variants.sh NAME "-DFLAG=V ..." ...
# Output: paper_1912_04822_b200/variants/NAME.so (load with GM_LIB=...).
set -e
cd "$(dirname "$0")/../paper_1912_04822_b200/csrc"
mkdir -p ../variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v --expt-relaxed-constexpr -I../../include \
    $flags -shared -o ../variants/$name.so abi.cu prepare.cu forward.cu backward.cu assemble.cu molc.cu pack.cu 2> ../variants/$name.log \
    || { grep -i error ../variants/$name.log; exit 1; }
  echo "$name: $(grep -A2 "${GREPK:-k_backward_index}" ../variants/$name.log | grep -E 'Used|spill' | tr '\n' ' ')"
done
