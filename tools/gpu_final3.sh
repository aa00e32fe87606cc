#!/bin/bash
O=gpurun_out/final
mkdir -p $O
timeout 900 python bench.py > $O/bench2.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py --quick > $O/sanitize_racecheck.log 2>&1; echo "rc=$?" >> $O/sanitize_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py --quick > $O/sanitize_synccheck.log 2>&1; echo "rc=$?" >> $O/sanitize_synccheck.log
true
