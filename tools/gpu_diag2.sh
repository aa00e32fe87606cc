mkdir -p gpurun_out
python tools/ab_libs.py _exp/r0.so _exp/v4.so _exp/pre2.so --strategy WD,HP --algo bfs --reps 3 --skewed > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/v4.so _exp/pre2.so --strategy WD --algo sssp --reps 5 >> gpurun_out/ab.log 2>&1
cp _exp/pre2.so paper_1711_00231_b200/libgraphlb_b200.so
timeout 600 python tools/profile_grid.py --strategy WD --algo sssp --loop graph > gpurun_out/grid_diag.log 2>&1
true
