mkdir -p gpurun_out
python tools/ab_libs.py _exp/nopol.so _exp/pol2.so --strategy WD,HP,BS,NS,EP --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/nopol.so _exp/pol2.so --strategy WD,HP,BS,NS,EP --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
true
