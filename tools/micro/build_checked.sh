#!/bin/bash
# The checked library (compute-sanitizer is closed on the GPU pool): every
# csrc/*.cu with -DPGC_CHECKED, so each PGC_DCHECK (pgc_internal.cuh) is a
# device assertion that prints and traps.  Loaded through
# PGC_LIB=tools/micro/libpgc_checked.so (tools/sanitize.py); never the product.
#   build_checked.sh [file.cu ...]   # only these files checked, the rest from build/pgc
set -e
cd "$(dirname "$0")/../.."
mkdir -p build/checked
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DPGC_CHECKED -I include"
if [ $# -gt 0 ]; then
  python -c "import sys; sys.path.insert(0, 'paper_2008_11321_b200'); import _build; _build.build()"
  OBJS=""
  for f in paper_2008_11321_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    if [[ " $* " == *" $b.cu "* ]]; then
      nvcc $FLAGS -c -o build/checked/$b.o $f; OBJS="$OBJS build/checked/$b.o"
    else
      OBJS="$OBJS build/pgc/$b.o"
    fi
  done
else
  pids=""
  OBJS=""
  for f in paper_2008_11321_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    nvcc $FLAGS -c -o build/checked/$b.o $f & pids="$pids $!"
    OBJS="$OBJS build/checked/$b.o"
  done
  for p in $pids; do wait $p; done
fi
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/micro/libpgc_checked.so $OBJS
echo tools/micro/libpgc_checked.so
