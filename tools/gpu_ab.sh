mkdir -p gpurun_out
python tools/ab_libs.py _exp/pipe2.so _exp/v3.so _exp/v4.so _exp/v4m3.so --strategy WD --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/pipe2.so _exp/v3.so _exp/v4.so _exp/v4m3.so --strategy WD --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
true
