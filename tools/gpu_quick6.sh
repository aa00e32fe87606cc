mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/suite.py --configs C3 --reps 2 > gpurun_out/suite_c3.log 2>&1
timeout 600 python tools/suite.py --configs C2,C4 --reps 3 > gpurun_out/suite_c2.log 2>&1
true
