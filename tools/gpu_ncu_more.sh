O=gpurun_out/ncu_more; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:k_wd_scan -s 1 -c 2 -o $O/wd_scan -f \
  python tools/profile_run.py --strategy WD --algo sssp --loop host --runs 1 > $O/wd_scan.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_hp_ -c 6 -o $O/hp_c4 -f \
  python tools/profile_run.py --strategy HP --algo bfs --loop host --runs 1 --skewed > $O/hp_c4.log 2>&1
true
