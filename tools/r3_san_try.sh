set -u
OUT=gpurun_out/san_try
mkdir -p $OUT
which compute-sanitizer > $OUT/which.txt 2>&1
timeout 300 compute-sanitizer --version >> $OUT/which.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize.py er --entries jp_adg > $OUT/memcheck_er.log 2>&1; echo "memcheck rc=$?" >> $OUT/status.txt
tail -20 $OUT/memcheck_er.log
