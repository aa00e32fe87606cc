#!/bin/bash
# Per-launch records for the headline run + a full ncu capture of the top relax kernel.
set -x
mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --strategy WD,BS,HP,EP,NS --algo sssp --runs 2 --loop host --records > gpurun_out/records_sssp.log 2>&1
timeout 300 python tools/profile_run.py --strategy WD,BS,HP,EP,NS --algo bfs --runs 2 --loop host --records > gpurun_out/records_bfs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wd_relax -s 3 -c 4 \
  -o gpurun_out/wd_relax -f python tools/profile_run.py --strategy WD --algo sssp --runs 1 --loop host > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wd_scan -s 3 -c 2 \
  -o gpurun_out/wd_scan -f python tools/profile_run.py --strategy WD --algo sssp --runs 1 --loop host > gpurun_out/ncu_scan.log 2>&1
true
