mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for algo in sssp bfs; do
  timeout 600 python tools/ab_libs.py _exp/head.so _exp/n24.so --strategy BS,EP,WD,NS,HP --algo $algo --scale 22 --reps 5 >> gpurun_out/ab24_s22.log 2>&1
done
timeout 900 python tools/ab_libs.py _exp/head.so _exp/n24.so --strategy WD,HP,BS --algo sssp --scale 24 --reps 3 >> gpurun_out/ab24_s24.log 2>&1
timeout 600 python tools/ab_libs.py _exp/head.so _exp/n24.so --strategy WD,HP,BS --algo bfs --scale 24 --reps 3 >> gpurun_out/ab24_s24.log 2>&1
true
