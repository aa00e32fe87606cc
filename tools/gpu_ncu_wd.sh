#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wd_relax -s 3 -c 3 \
  -o gpurun_out/wd_relax2 -f python tools/profile_run.py --strategy WD --algo sssp --runs 1 --loop host > gpurun_out/ncu_full.log 2>&1
true
