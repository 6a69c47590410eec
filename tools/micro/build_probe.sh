#!/bin/bash
# Build the instrumented (PGC_PROBE) variant of libpgc for tools/micro/hop_probe.py.
set -e
cd "$(dirname "$0")/../.."
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  -DPGC_PROBE -I include -o tools/micro/libpgc_probe.so paper_2008_11321_b200/csrc/*.cu
