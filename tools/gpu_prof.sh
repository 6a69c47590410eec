#!/bin/bash
# One profiling pass (run under gpurun): plain run, ncu launch list, ncu --set full
# of the top kernels.  Usage: TAG=r1b tools/gpu_prof.sh
set -u
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
CMD="python bench.py --quick --steps 1 --warmup 3 ${BENCH_EXTRA:-}"
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_jp_color}" -s ${KSKIP:-3} -c ${KCOUNT:-1} -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo "rc=$?"
tail -2 $OUT/plain.log | cut -c1-400
