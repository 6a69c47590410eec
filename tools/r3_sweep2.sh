#!/bin/bash
# ADG-M launch list (ncu) + JP-R backoff sweep.  Logs under gpurun_out/$TAG.
set -u
OUT=gpurun_out/${TAG:-sw2}
mkdir -p $OUT
run() {  # method tune
  F=$OUT/bench_$1_${2//[=,]/_}.json
  PGC_TUNE=$2 timeout 600 python bench.py --method $1 --no-e2e --no-cpu-baseline --steps ${STEPS:-5} --warmup 3 > $F.log 2>&1
  echo "bench $1 $2 rc=$?" >> $OUT/status.txt
  tail -1 $F.log > $F
  python -c "import json; d=json.load(open('$F')); print('$1 $2', round(d['ms_per_step'],3), d.get('breakdown_ms'))" >> $OUT/summary.txt 2>&1
}
for T in jp_light_sleep_max=8192 jp_light_sleep_max=1024 jp_light_sleep_max=256 jp_heavy_sleep_max=64 jp_heavy_warps=2 jp_heavy_warps=3; do run jp-r $T; done
CMD="python bench.py --method jp-adg-m --quick --serial-schedule --steps 1 --warmup 3"
$CMD > $OUT/m_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_adgm.csv $CMD > $OUT/ncu_m.log 2>&1
echo "ncu adg-m rc=$?" >> $OUT/status.txt
cat $OUT/status.txt $OUT/summary.txt
