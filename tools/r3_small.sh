set -u
OUT=gpurun_out/r3_small
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_small.py -q -x --timeout 600 > $OUT/pytest_small.log 2>&1; echo "small rc=$?" >> $OUT/status.txt
tail -5 $OUT/pytest_small.log
for W in er:1/10 grid:1/10; do
  C=${W%%:*}; E=${W##*:}
  timeout 600 python bench.py --config $C --eps $E --no-cpu-baseline > $OUT/bench_$C.log 2>&1; echo "bench $C rc=$?" >> $OUT/status.txt
  tail -1 $OUT/bench_$C.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['small_path'], d['breakdown_ms'], d['roofline']['frac'])"
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
tail -3 $OUT/pytest_gpu.log
cat $OUT/status.txt
