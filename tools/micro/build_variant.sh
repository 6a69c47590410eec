#!/bin/bash
# Build an A/B variant of libpgc with extra -D flags: build_variant.sh <name> -DFOO ...
# (loaded through PGC_LIB=tools/micro/libpgc_<name>.so; never the product library)
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  "$@" -I include -o tools/micro/libpgc_$name.so paper_2008_11321_b200/csrc/*.cu
