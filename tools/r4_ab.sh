#!/bin/bash
# A/B of library tuning knobs on one box: headline bench per variant (PGC_TUNE).
#   TAG=r4_pipe VARIANTS="filter_pipe=0 filter_pipe=1" [CONFIG=rmat24 EPS=1/10] tools/r4_ab.sh
set -u
OUT=gpurun_out/${TAG:-r4_ab}
mkdir -p $OUT
for V in ${VARIANTS:-"filter_pipe=0 filter_pipe=1"}; do
  F=$OUT/bench_${CONFIG:-rmat24}_${V//[=,]/_}.json
  PGC_TUNE=$V timeout 900 python bench.py --config ${CONFIG:-rmat24} --eps ${EPS:-1/10} --no-e2e ${BENCH_ARGS:-} > $F.log 2>&1
  echo "bench $V rc=$?" >> $OUT/status.txt
  tail -1 $F.log > $F
  python - "$F" "$V" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], 'ms/step', round(d['ms_per_step'],3), 'median', round(d['timing']['median_ms'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()}, d.get('parity'))
PY
done
cat $OUT/status.txt
