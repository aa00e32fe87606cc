mkdir -p gpurun_out
python tools/ab_libs.py _exp/head.so _exp/hpsplit.so --strategy HP --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/head.so _exp/hpsplit.so --strategy HP --algo bfs --reps 3 --skewed >> gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/head.so _exp/hpsplit.so --strategy HP --algo sssp --reps 3 --skewed >> gpurun_out/ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
true
