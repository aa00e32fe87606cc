mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py _exp/c_bf5d3cb.so _exp/c_78c1270.so _exp/c_cc98f1f.so _exp/c_b6b28f4.so _exp/c_8cc8fb8.so _exp/head.so _exp/cur.so --strategy WD --algo sssp --reps 7 > gpurun_out/bisect.log 2>&1
timeout 900 python tools/ab_libs.py _exp/c_bf5d3cb.so _exp/c_78c1270.so _exp/c_cc98f1f.so _exp/c_b6b28f4.so _exp/c_8cc8fb8.so _exp/head.so _exp/cur.so --strategy WD --algo bfs --reps 7 >> gpurun_out/bisect.log 2>&1
true
