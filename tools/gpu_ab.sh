mkdir -p gpurun_out
python tools/ab_libs.py _exp/keep.so _exp/dense.so --strategy WD --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/keep.so _exp/dense.so --strategy WD --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/keep.so _exp/dense.so --strategy WD --algo sssp --reps 3 --skewed >> gpurun_out/ab.log 2>&1
cp _exp/dense.so paper_1711_00231_b200/libgraphlb_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_run.py --strategy WD --algo sssp --runs 2 --loop host --records > gpurun_out/records.log 2>&1
true
