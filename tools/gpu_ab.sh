mkdir -p gpurun_out
python tools/ab_libs.py _exp/base.so _exp/minb4.so _exp/minb2.so --strategy WD,HP --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
GLB_L2_PERSIST=1 python tools/ab_libs.py _exp/base.so _exp/minb4.so --strategy WD --algo sssp --reps 5 > gpurun_out/ab_l2.log 2>&1
python tools/ab_libs.py _exp/base.so _exp/minb4.so --strategy WD,HP --algo bfs --reps 5 > gpurun_out/ab_bfs.log 2>&1
true
