mkdir -p gpurun_out
python tools/ab_libs.py _exp/c8.so _exp/c16.so _exp/c8e8.so --strategy WD,BS,HP --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/c8.so _exp/c16.so _exp/c8e8.so --strategy WD,BS --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
true
