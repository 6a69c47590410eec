#!/bin/bash
# One GPU pass: build, smoke, gpu tests, short bench.  Logs under gpurun_out/.
set -u
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q --timeout 600 ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
tail -3 $OUT/bench.log
