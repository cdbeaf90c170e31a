#!/bin/bash
# Build librebk variants with extra -D flags into tools/librebk_<name>.so
# (A/B experiments through REBK_LIB).  usage: tools/build_variants.sh name "-DFOO -DBAR" ...
# The source list is the product build's (paper_2001_04179_b200/build.py).
set -e
cd "$(dirname "$0")/.."
C=paper_2001_04179_b200/csrc
SRC=$(python -c "from paper_2001_04179_b200.build import SOURCES; print(' '.join('$C/' + s for s in SOURCES))")
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -ldl $flags \
    $SRC -o tools/librebk_$name.so &
done
wait
