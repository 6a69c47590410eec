#!/bin/bash
# Round-2 evidence pass (run under gpurun, one GPU):
#  1. bench.py on all 8 (graph, eps) runs of the five BASELINE configs
#     (each line: cpu_baseline, in-run parity, J, d, T, K),
#  2. per-workload UPDATE DRAM traffic (ncu dram bytes; tools/traffic.py),
#  3. ncu --set full of the top kernels on R-MAT 24 (round 1's k_update_light,
#     two k_update_heavy_f rounds, the JP core + bulk),
#  4. the ncu launch list of the headline bench command.
#   TAG=r2_a STAGES="bench traffic full launches" tools/r2_profile.sh  -> gpurun_out/$TAG/
# Every command runs plain (exit 0) before it runs under ncu (B200_PROFILING.md).
set -u
OUT=gpurun_out/${TAG:-r2_prof}
mkdir -p $OUT
STAGES=${STAGES:-"bench traffic full launches"}
nvidia-smi > $OUT/smi.txt 2>&1
WL="er:1/10 rmat20:1/100 rmat20:1/10 rmat20:1/2 grid:1/10 rmat24:1/10 cl:1/100 cl:1/2"
for S in $STAGES; do
case $S in
bench)
  for W in ${BENCH_WL:-$WL}; do
    C=${W%%:*}; E=${W##*:}; F=$OUT/bench_${C}_${E/\//_}.json
    timeout 900 python bench.py --config $C --eps $E ${BENCH_ARGS:-} > $F.log 2>&1
    echo "bench $W rc=$?" >> $OUT/status.txt
    tail -1 $F.log > $F
  done ;;
traffic)
  for W in ${TRAFFIC_WL:-$WL}; do
    C=${W%%:*}; E=${W##*:}; F=$OUT/traffic_${C}_${E/\//_}.csv
    timeout 600 python tools/traffic.py run --config $C --eps $E > /dev/null 2>&1 && \
    timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:k_update --csv --log-file $F python tools/traffic.py run --config $C --eps $E > $OUT/traffic.log 2>&1
    echo "traffic $W rc=$?" >> $OUT/status.txt
  done ;;
full)
  python tools/launch_times.py > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_update_light -s 8 -c 1 -o $OUT/upd_light_r1 python tools/launch_times.py > $OUT/f1.log 2>&1
  echo "full light rc=$?" >> $OUT/status.txt
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_update_heavy_f -s 10 -c 2 -o $OUT/upd_heavy_f python tools/launch_times.py > $OUT/f2.log 2>&1
  echo "full heavy_f rc=$?" >> $OUT/status.txt
  python tools/launch_times.py jp_split_overlap=0 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_jp_core|k_jp_bulk" -s 2 -c 2 -o $OUT/jp python tools/launch_times.py jp_split_overlap=0 > $OUT/f3.log 2>&1
  echo "full jp rc=$?" >> $OUT/status.txt ;;
launches)
  CMD="python bench.py --quick --serial-schedule --steps 1 --warmup 3"
  $CMD > $OUT/plain_quick.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
  echo "launches rc=$?" >> $OUT/status.txt ;;
checked)
  # compute-sanitizer is closed on this pool: the checked library instead
  # (device bounds asserts, workspace canaries, poisoned workspace and outputs)
  for G in ${CHK_GRAPHS:-er rmat16 grid rmat20}; do
    PGC_LIB=tools/micro/libpgc_checked.so timeout 900 python tools/sanitize.py $G > $OUT/checked_$G.log 2>&1
    echo "checked $G rc=$?" >> $OUT/status.txt
    CUDA_LAUNCH_BLOCKING=1 PGC_LIB=tools/micro/libpgc_checked.so timeout 900 python tools/sanitize.py $G > $OUT/checked_blocking_$G.log 2>&1
    echo "checked blocking $G rc=$?" >> $OUT/status.txt
    PGC_LIB=tools/micro/libpgc_checked.so timeout 900 python tools/sanitize.py $G --serial > $OUT/checked_serial_$G.log 2>&1
    echo "checked serial $G rc=$?" >> $OUT/status.txt
  done
  PGC_LIB=tools/micro/libpgc_checked.so timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/checked_pytest.log 2>&1
  echo "checked pytest rc=$?" >> $OUT/status.txt ;;
esac
done
cat $OUT/status.txt
