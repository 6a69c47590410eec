#!/bin/bash
# Build the instrumented (PGC_PROBE) variant of libpgc for tools/micro/core_probe.py:
# jp.cu (the only file PGC_PROBE changes) with -DPGC_PROBE, linked with the
# product objects of the other files (build/pgc, from paper_2008_11321_b200/_build.py).
set -e
cd "$(dirname "$0")/../.."
python -c "import sys; sys.path.insert(0, 'paper_2008_11321_b200'); import _build; _build.build()"
mkdir -p build/probe
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -c \
  -DPGC_PROBE -I include -o build/probe/jp.o paper_2008_11321_b200/csrc/jp.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/micro/libpgc_probe.so \
  $(ls build/pgc/*.o | grep -v '/jp.o$') build/probe/jp.o
