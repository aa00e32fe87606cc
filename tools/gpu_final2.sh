#!/bin/bash
O=gpurun_out/final
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_host.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --e2e-steps 0 --loop host > $O/ncu_launch_bench_host.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > $O/sanitize_memcheck.log 2>&1; echo "rc=$?" >> $O/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py > $O/sanitize_racecheck.log 2>&1; echo "rc=$?" >> $O/sanitize_racecheck.log
true
