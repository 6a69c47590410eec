#!/bin/bash
# libpgc with the one-kernel small path built with -DPGC_PROBE (phase timeline
# printed by the kernel); the other objects from build/pgc.  Never the product.
set -e
cd "$(dirname "$0")/../.."
python -c "import sys; sys.path.insert(0, 'paper_2008_11321_b200'); import _build; _build.build()"
mkdir -p build/probe
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -c \
  -DPGC_PROBE -I include -o build/probe/small.o paper_2008_11321_b200/csrc/small.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/micro/libpgc_small_probe.so \
  $(ls build/pgc/*.o | grep -v '/small.o$') build/probe/small.o
