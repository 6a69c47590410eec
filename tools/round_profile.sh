#!/bin/bash
# Round profile (run under gpurun, one GPU): the bench line, the ncu launch list
# of the same bench command, DRAM bytes of every UPDATE launch of one step per
# workload (bench.py's roofline `traffic`, merged into profiles/traffic.json by
# tools/traffic.py parse), and ncu --set full of the top kernels.
#   TAG=r2_a tools/round_profile.sh   -> gpurun_out/$TAG/
# Every command runs plain (exit 0) before it runs under ncu (B200_PROFILING.md).
set -u
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi > $OUT/smi.txt 2>&1
python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" > $OUT/status.txt
# ncu serialises kernels: profile the one-stream schedule (same kernels, see bench.py)
CMD="python bench.py --quick --serial-schedule --steps 1 --warmup 3"
$CMD > $OUT/plain_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
# UPDATE DRAM traffic per workload (two calls; the second is the measured one)
for W in ${TRAFFIC:-rmat24:1/10}; do
  C=${W%%:*}; E=${W##*:}; F=$OUT/traffic_${C}_${E/\//_}.csv
  python tools/traffic.py run --config $C --eps $E > /dev/null 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_update --csv --log-file $F python tools/traffic.py run --config $C --eps $E > $OUT/traffic.log 2>&1
  echo "traffic $W rc=$?" >> $OUT/status.txt
done
# full sets: round 1's light UPDATE, the two biggest filtered heavy rounds (3, 4), the JP kernels
python tools/launch_times.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_light -s 8 -c 1 -o $OUT/upd_light_r1 python tools/launch_times.py > $OUT/f1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_heavy_f -s 10 -c 2 -o $OUT/upd_heavy_f python tools/launch_times.py > $OUT/f2.log 2>&1
python tools/launch_times.py jp_split_overlap=0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_jp_core|k_jp_bulk" -s 2 -c 2 -o $OUT/jp python tools/launch_times.py jp_split_overlap=0 > $OUT/f3.log 2>&1
echo "full rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
