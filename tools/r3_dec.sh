#!/bin/bash
# DEC-ADG-ITR pass-grid sweep + mega sweep on JP-R.  Logs under gpurun_out/$TAG.
set -u
OUT=gpurun_out/${TAG:-dec}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "${PYK:-dec_adg or mega}" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
run() {  # method tune
  F=$OUT/bench_$1_${2//[=,]/_}.json
  PGC_TUNE=$2 timeout 600 python bench.py --method $1 --no-e2e --no-cpu-baseline --steps ${STEPS:-5} --warmup 3 > $F.log 2>&1
  echo "bench $1 $2 rc=$?" >> $OUT/status.txt
  tail -1 $F.log > $F
  python -c "import json; d=json.load(open('$F')); print('$1 $2', round(d['ms_per_step'],3), d.get('breakdown_ms',{}).get('jp'))" >> $OUT/summary.txt 2>&1
}
for T in ${DEC_TUNES:-itr_members_per_warp=4 itr_members_per_warp=1 itr_members_per_warp=2 itr_members_per_warp=16}; do run dec-adg-itr $T; done
for T in ${MEGA_TUNES:-jp_mega_pred=2048 jp_mega_pred=512,jp_mega_chunk=256 jp_mega_pred=1024,jp_mega_chunk=512 jp_mega_pred=4096 jp_mega_pred=2048,jp_mega_chunk=384}; do run jp-r $T; done
cat $OUT/status.txt $OUT/summary.txt
