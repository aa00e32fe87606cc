mkdir -p gpurun_out
for v in 0 1 2; do
  if [ $v = 0 ]; then unset GLB_WD_SKIP; else export GLB_WD_SKIP=$v; fi
  echo "== GLB_WD_SKIP=$v" >> gpurun_out/skip_suite.log
  timeout 300 python tools/suite.py --configs C2,C4 --tags WD --algos sssp --reps 5 >> gpurun_out/skip_suite.log 2>&1
done
export GLB_WD_SKIP=1
timeout 1500 python -m pytest tests -m gpu -x -q -k "corpus or random" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
true
