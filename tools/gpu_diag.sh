mkdir -p gpurun_out
timeout 600 python tools/profile_grid.py --strategy WD --algo sssp --loop host > gpurun_out/grid_diag.log 2>&1
timeout 600 python tools/profile_grid.py --strategy WD --algo sssp --loop graph >> gpurun_out/grid_diag.log 2>&1
timeout 600 python tools/profile_grid.py --strategy BS --algo sssp --loop graph >> gpurun_out/grid_diag.log 2>&1
timeout 300 python tools/profile_run.py --strategy HP --algo bfs --skewed --runs 2 --loop host --records > gpurun_out/hp_c4.log 2>&1
python tools/ab_libs.py _exp/v4.so _exp/fused.so --strategy WD --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/v4.so _exp/fused.so --strategy WD --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
true
