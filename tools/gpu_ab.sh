mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "corpus or random or hp or c1 or dist_bits" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/ab_libs.py _exp/hpbig.so _exp/hpbig3.so --strategy HP --algo bfs --reps 5 --skewed > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/hpbig.so _exp/hpbig3.so --strategy HP --algo sssp --reps 5 --skewed >> gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/hpbig.so _exp/hpbig3.so --strategy HP --algo sssp --reps 5 >> gpurun_out/ab.log 2>&1
true
