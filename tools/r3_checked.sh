# Checked runs (compute-sanitizer is closed on the pool): every entry point
# on configs 1-3 plus an R-MAT 16, with the checked library (device bounds /
# invariant asserts), normal / CUDA_LAUNCH_BLOCKING / one-stream schedules,
# then the GPU test suite on the checked library.
set -u
OUT=gpurun_out/${TAG:-r3_checked}
mkdir -p $OUT
L=tools/micro/libpgc_checked.so
for G in ${CHK_GRAPHS:-er rmat16 grid rmat20}; do
  PGC_LIB=$L timeout 900 python tools/sanitize.py $G > $OUT/checked_$G.log 2>&1
  echo "checked $G rc=$?" >> $OUT/status.txt
  CUDA_LAUNCH_BLOCKING=1 PGC_LIB=$L timeout 900 python tools/sanitize.py $G > $OUT/checked_blocking_$G.log 2>&1
  echo "checked blocking $G rc=$?" >> $OUT/status.txt
  PGC_LIB=$L timeout 900 python tools/sanitize.py $G --serial > $OUT/checked_serial_$G.log 2>&1
  echo "checked serial $G rc=$?" >> $OUT/status.txt
done
PGC_LIB=$L timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > $OUT/checked_pytest.log 2>&1
echo "checked pytest rc=$?" >> $OUT/status.txt
tail -3 $OUT/checked_pytest.log
cat $OUT/status.txt
