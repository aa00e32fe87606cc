mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --strategy HP,WD --algo bfs --skewed --runs 2 --loop host --records > gpurun_out/hp_c4.log 2>&1
true
