mkdir -p gpurun_out
python tools/ab_libs.py _exp/dense.so _exp/hpw2.so _exp/hpw2m2.so --strategy HP --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/dense.so _exp/hpw2.so _exp/hpw2m2.so --strategy HP --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/dense.so _exp/hpw2.so _exp/hpw2m2.so --strategy HP --algo sssp --reps 3 --skewed >> gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/dense.so _exp/hpw2.so _exp/hpw2m2.so --strategy HP --algo bfs --reps 3 --skewed >> gpurun_out/ab.log 2>&1
cp _exp/hpw2.so paper_1711_00231_b200/libgraphlb_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
true
