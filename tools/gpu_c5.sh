mkdir -p gpurun_out
free -g > gpurun_out/free.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1800 python tools/suite.py --configs C5 --reps 1 --tags WD,BS,EP,NS,HP --out gpurun_out/suite_c5.json > gpurun_out/suite_c5.log 2>&1; echo "rc=$?" >> gpurun_out/suite_c5.log
true
