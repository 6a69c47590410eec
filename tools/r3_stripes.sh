#!/bin/bash
# Heavy ticket stripes: parity, then JP-ADG / JP-R bench per stripe count.
set -u
OUT=gpurun_out/${TAG:-stripes}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "stripes or mega" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
run() {  # method tune
  F=$OUT/bench_$1_${2//[=,]/_}.json
  PGC_TUNE=$2 timeout 600 python bench.py --method $1 --no-e2e --no-cpu-baseline --steps ${STEPS:-10} --warmup 3 > $F.log 2>&1
  echo "bench $1 $2 rc=$?" >> $OUT/status.txt
  tail -1 $F.log > $F
  python -c "import json; d=json.load(open('$F')); b=d.get('breakdown_ms'); print('$1 $2', round(d['ms_per_step'],3), round(b['core'],3), round(b['jp'],3))" >> $OUT/summary.txt 2>&1
}
for T in jp_heavy_stripes=1 jp_heavy_stripes=2 jp_heavy_stripes=4 jp_heavy_stripes=8 jp_heavy_stripes=1; do run jp-adg $T; done
for T in jp_heavy_stripes=1 jp_heavy_stripes=4 jp_heavy_stripes=8; do run jp-r $T; done
cat $OUT/status.txt $OUT/summary.txt
