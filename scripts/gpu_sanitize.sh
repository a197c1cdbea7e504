# compute-sanitizer memcheck / synccheck / racecheck over scripts/sanitize.py
set -x
timeout 300 python scripts/sanitize.py 2>&1 | tail -1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/san_memcheck.log 2>&1; tail -2 gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py > gpurun_out/san_synccheck.log 2>&1; tail -2 gpurun_out/san_synccheck.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python scripts/sanitize.py > gpurun_out/san_racecheck.log 2>&1; tail -3 gpurun_out/san_racecheck.log
