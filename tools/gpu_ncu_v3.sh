mkdir -p gpurun_out
./_exp/gather_peak 22 26 > gpurun_out/gather_peak.log 2>&1
./_exp/gather_peak 24 26 >> gpurun_out/gather_peak.log 2>&1
cp _exp/v3.so paper_1711_00231_b200/libgraphlb_b200.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wd_relax -s 3 -c 2 \
  -o gpurun_out/wd_relax3 -f python tools/profile_run.py --strategy WD --algo sssp --runs 1 --loop host > gpurun_out/ncu_full.log 2>&1
true
