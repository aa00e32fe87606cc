# full GPU tier + suite C2/C3/C4 on the id-ordered-frontier build
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 1500 python tools/suite.py --configs C2,C4,C3 --reps 3 --out gpurun_out/suite.json > gpurun_out/suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite.log
grep "^|" gpurun_out/suite.log | tail -n 30
