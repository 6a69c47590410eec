#!/bin/bash
# Round-2 final evidence (one GPU, under gpurun):
#   bench   all 8 (graph, eps) runs of the five configs (cpu_baseline, parity, J, d)
#   methods the §8(f) rows on R-MAT 24 (bench.py --method ...)
#   traffic per-workload DRAM bytes of the dominant kernel(s) (UPDATE, or the
#           one-kernel path's kernel on ER / the grid)
#   launches ncu launch list of the headline bench command
#   full    ncu --set full: round 1's k_update_light, two k_update_heavy_f rounds,
#           the JP core + bulk, k_small_jp_adg (grid), k_tiny_jp_adg (ER)
#   TAG=r2_final STAGES="traffic bench methods launches full" tools/r2_final.sh
# (traffic first: bench.py reads the measured bytes from profiles/traffic.json)
set -u
OUT=gpurun_out/${TAG:-r2_final}
mkdir -p $OUT
STAGES=${STAGES:-"traffic bench methods launches full"}
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
methods)
  for M in ${METHODS:-jp-adg-o jp-adg-m dec-adg-itr jp-r jp-ff jp-lf jp-llf adg-push adg-pull}; do
    F=$OUT/bench_method_$M.json
    timeout 900 python bench.py --method $M --no-e2e > $F.log 2>&1
    echo "method $M rc=$?" >> $OUT/status.txt
    tail -1 $F.log > $F
  done ;;
traffic)
  for W in ${TRAFFIC_WL:-rmat20:1/100 rmat20:1/10 rmat20:1/2 rmat24:1/10 cl:1/100 cl:1/2}; do
    C=${W%%:*}; E=${W##*:}; F=$OUT/traffic_${C}_${E/\//_}.csv
    timeout 600 python tools/traffic.py run --config $C --eps $E > /dev/null 2>&1 && \
    timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:k_update --csv --log-file $F python tools/traffic.py run --config $C --eps $E > $OUT/traffic.log 2>&1
    echo "traffic $W rc=$?" >> $OUT/status.txt
    python tools/traffic.py parse $F --workload $C-eps$E --source profiles/${TAG:-r2_final}/$(basename $F) >> $OUT/traffic_parse.log 2>&1
  done
  for W in ${TRAFFIC_SMALL_WL:-er:1/10 grid:1/10}; do
    C=${W%%:*}; E=${W##*:}; F=$OUT/traffic_${C}_${E/\//_}_small.csv
    timeout 600 python tools/traffic.py run --config $C --eps $E > /dev/null 2>&1 && \
    timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:"k_small|k_tiny" --csv --log-file $F python tools/traffic.py run --config $C --eps $E > $OUT/traffic_small.log 2>&1
    echo "traffic small $W rc=$?" >> $OUT/status.txt
    KN=k_tiny_jp_adg; grep -q k_small_jp_adg $F && KN=k_small_jp_adg
    python tools/traffic.py parse $F --kernel $KN --workload $C-eps$E-small --source profiles/${TAG:-r2_final}/$(basename $F) >> $OUT/traffic_parse.log 2>&1
  done
  cp profiles/traffic.json $OUT/traffic.json ;;
launches)
  CMD="python bench.py --quick --serial-schedule --steps 1 --warmup 3"
  $CMD > $OUT/plain_quick.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
  echo "launches rc=$?" >> $OUT/status.txt ;;
full)
  python tools/launch_times.py > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_update_light -s 8 -c 1 -o $OUT/upd_light_r1 python tools/launch_times.py > $OUT/f1.log 2>&1
  echo "full light rc=$?" >> $OUT/status.txt
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_update_heavy_f -s 10 -c 2 -o $OUT/upd_heavy_f python tools/launch_times.py > $OUT/f2.log 2>&1
  echo "full heavy_f rc=$?" >> $OUT/status.txt
  python tools/launch_times.py jp_split_overlap=0 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_jp_core|k_jp_bulk" -s 3 -c 2 -o $OUT/jp python tools/launch_times.py jp_split_overlap=0 > $OUT/f3.log 2>&1
  echo "full jp rc=$?" >> $OUT/status.txt
  timeout 600 python tools/traffic.py run --config grid > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_small -s 1 -c 1 -o $OUT/small_grid python tools/traffic.py run --config grid > $OUT/f4.log 2>&1
  echo "full small grid rc=$?" >> $OUT/status.txt
  timeout 600 python tools/traffic.py run --config er > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiny -s 1 -c 1 -o $OUT/tiny_er python tools/traffic.py run --config er > $OUT/f5.log 2>&1
  echo "full tiny er rc=$?" >> $OUT/status.txt ;;
esac
done
cat $OUT/status.txt
