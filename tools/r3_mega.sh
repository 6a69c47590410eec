#!/bin/bash
# Mega-vertex chunks in the JP bulk: parity tests, then JP-R / JP-FF / JP-ADG
# bench lines per (jp_mega_pred, jp_mega_chunk).  Logs under gpurun_out/$TAG.
set -u
OUT=gpurun_out/${TAG:-mega}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "${PYK:-mega or baselines or heavy_paths or config_parity}" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
for M in ${METHODS:-jp-r jp-ff jp-adg}; do
  for T in ${TUNES:-jp_mega_pred=0 jp_mega_pred=2048,jp_mega_chunk=1024 jp_mega_pred=2048,jp_mega_chunk=512 jp_mega_pred=1024,jp_mega_chunk=256}; do
    F=$OUT/bench_${M}_${T//[=,]/_}.json
    PGC_TUNE=$T timeout 600 python bench.py --method $M --no-e2e --no-cpu-baseline --steps ${STEPS:-5} --warmup 3 > $F.log 2>&1
    echo "bench $M $T rc=$?" >> $OUT/status.txt
    tail -1 $F.log > $F
    python -c "import json; d=json.load(open('$F')); print('$M $T', round(d['ms_per_step'],3), d.get('breakdown_ms',{}).get('jp'), d.get('parity'))" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/status.txt $OUT/summary.txt
