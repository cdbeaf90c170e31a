#!/bin/bash
# Build librebk variants with extra -D flags into tools/librebk_<name>.so
# (A/B experiments through REBK_LIB).  usage: tools/build_variants.sh name "-DFOO -DBAR" ...
set -e
cd "$(dirname "$0")/.."
C=paper_2001_04179_b200/csrc
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -ldl $flags \
    $C/rebk_dense.cu $C/rebk_dense_fast.cu $C/rebk_dense_split.cu $C/rebk_dense_stream.cu $C/rebk_csr.cu $C/rebk_mrhs.cu $C/rebk_mrhs_tc.cu $C/rebk_shard.cu $C/rebk_beta.cu $C/rebk_nccl.cu \
    $C/rebk_api.cu -o tools/librebk_$name.so &
done
wait
