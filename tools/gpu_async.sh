mkdir -p gpurun_out
for algo in sssp bfs; do
  timeout 600 python tools/ab_libs.py _exp/base2.so _exp/async.so --strategy WD,HP --algo $algo --reps 7 >> gpurun_out/async_s22.log 2>&1
  timeout 600 python tools/ab_libs.py _exp/base2.so _exp/async.so --strategy WD,HP --algo $algo --reps 5 --skewed >> gpurun_out/async_s22.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/ab_records.py _exp/base2.so _exp/async.so --strategy WD --algo sssp > gpurun_out/async_rec.log 2>&1
true
