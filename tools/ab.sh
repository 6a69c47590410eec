#!/bin/bash
# A/B: run tools/sweep.py on the product library and on each named variant
# (tools/micro/libpgc_<name>.so).  Usage: tools/ab.sh "<sweep args>" name1 name2 ...
args=$1; shift
echo "== product"; python tools/sweep.py $args
for v in "$@"; do echo "== $v"; PGC_LIB=tools/micro/libpgc_$v.so python tools/sweep.py $args; done
