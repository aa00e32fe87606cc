mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
true
